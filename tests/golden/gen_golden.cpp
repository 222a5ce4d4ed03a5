// gen_golden.cpp -- golden-vector generator (test infrastructure, run only in the
// build container where /root/reference exists; its OUTPUT is committed).
//
// Re-creates the reference's own known-answer inputs -- the std::mt19937_64 +
// libstdc++-distribution sequences of proj/tests/test_expact.cpp,
// proj/tests/test_stencil.cpp and proj/tests/acceptance.cpp -- through the
// reference's public API and its test header proj/tests/oracles.hpp (included
// from /root/reference, not copied), and records inputs, the reference library's
// outputs and the dense-oracle outputs.  Output: a flat record stream read by
// make_golden.py:  [u32 name_len][name][u8 kind: 0=f64 1=i64 2=i32][u64 count][payload].
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "gliosim/errors.hpp"
#include "gliosim/expact.hpp"
#include "gliosim/integrator.hpp"
#include "gliosim/sparse.hpp"
#include "gliosim/stencil.hpp"
#include "oracles.hpp"

namespace {

FILE* g_out = nullptr;

void put(const std::string& name, int kind, const void* data, uint64_t count, size_t elem) {
    uint32_t len = static_cast<uint32_t>(name.size());
    uint8_t k = static_cast<uint8_t>(kind);
    std::fwrite(&len, 4, 1, g_out);
    std::fwrite(name.data(), 1, len, g_out);
    std::fwrite(&k, 1, 1, g_out);
    std::fwrite(&count, 8, 1, g_out);
    if (count) std::fwrite(data, elem, count, g_out);
}
void putd(const std::string& n, const std::vector<double>& v) { put(n, 0, v.data(), v.size(), 8); }
void putd(const std::string& n, double x) { put(n, 0, &x, 1, 8); }
void puti(const std::string& n, const std::vector<int64_t>& v) { put(n, 1, v.data(), v.size(), 8); }
void puti(const std::string& n, int64_t x) { put(n, 1, &x, 1, 8); }
void put32(const std::string& n, const std::vector<int32_t>& v) { put(n, 2, v.data(), v.size(), 4); }

void put_csr(const std::string& p, const gliosim::SparseOperator& a) {
    puti(p + ".dim", a.dim());
    puti(p + ".offs", a.row_offsets());
    put32(p + ".cols", a.column_indices());
    putd(p + ".vals", a.coefficients());
    putd(p + ".norm1", a.one_norm());
}

// test_expact.cpp:79-96 and :146-175 (same generator calls, same order).
void random_operator_kats(const char* tag, uint64_t seed, int lo, int hi, double tlo, double thi, int trials,
                          double tol, bool phi, bool loop_until_done) {
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> size(lo, hi);
    std::uniform_real_distribution<double> target(tlo, thi);
    int done = 0, trial = 0;
    while (loop_until_done ? done < trials : trial < trials) {
        const int n = size(rng);
        const gliosim::SparseOperator a = oracles::random_sparse(rng, n, 0.3);
        if (a.one_norm() == 0.0) {
            ++trial;
            continue;
        }
        const int idx = loop_until_done ? done : trial;
        const double sign = (idx % 2 == 0) ? 1.0 : -1.0;
        const double t = sign * target(rng) / a.one_norm();
        const std::vector<double> b = oracles::random_vector(rng, n);
        const std::string p = std::string(tag) + "." + std::to_string(done);
        put_csr(p + ".A", a);
        putd(p + ".t", t);
        putd(p + ".tol", tol);
        putd(p + ".b", b);
        const oracles::Dense dense = oracles::scale(oracles::dense_from_sparse(a), t);
        if (phi) {
            putd(p + ".ref", gliosim::phi1v(t, a, b, tol));
            putd(p + ".dense", oracles::apply(oracles::phi1(dense), b));
            std::vector<double> e = oracles::apply(oracles::expm(dense), b);
            putd(p + ".dense_exp", e);
        } else {
            putd(p + ".ref", gliosim::expmv(t, a, b, tol));
            putd(p + ".dense", oracles::apply(oracles::expm(dense), b));
        }
        if (loop_until_done && phi) putd(p + ".ref_exp", gliosim::expmv(t, a, b, tol));
        ++done;
        ++trial;
    }
    puti(std::string(tag) + ".count", done);
}

// test_stencil.cpp:41-48 random_field and the grids of :54-69.
void stencil_kats() {
    const gliosim::Grid grids[] = {gliosim::Grid(4, 3, 2, 2.0), gliosim::Grid(5, 4, 1, 0.7), gliosim::Grid(7, 1, 1, 1.3),
                                   gliosim::Grid(9, 7, 6, 1.1)};
    uint64_t seed = 41;
    int idx = 0;
    for (const gliosim::Grid& g : grids) {
        for (double zero_frac : {0.0, 0.35}) {
            std::mt19937_64 rng(++seed);
            std::uniform_real_distribution<double> coef(0.01, 0.2);
            std::uniform_real_distribution<double> pick(0.0, 1.0);
            gliosim::DiffusionField d(g);
            for (double& x : d.d) x = (pick(rng) < zero_frac) ? 0.0 : coef(rng);
            const gliosim::SparseOperator a = gliosim::assemble_diffusion(d);
            std::uniform_real_distribution<double> val(-1.0, 1.0);
            std::vector<double> x(static_cast<size_t>(g.num_points()));
            for (double& v : x) v = val(rng);
            const std::string p = "stencil." + std::to_string(idx++);
            puti(p + ".shape", std::vector<int64_t>{g.nx, g.ny, g.nz});
            putd(p + ".h", g.h);
            putd(p + ".d", d.d);
            putd(p + ".x", x);
            putd(p + ".Ax", a.apply(x));
            put_csr(p + ".A", a);
            // pure-diffusion step = expmv (test_integrator.cpp:81-97 shape)
            std::vector<double> u(x.size());
            for (size_t i = 0; i < u.size(); ++i) u[i] = 0.5 + 0.5 * x[i];
            putd(p + ".u", u);
            putd(p + ".step_rho0", gliosim::step(a, u, 0.0, 12.0, 1e-10));
            putd(p + ".step_rho", gliosim::step(a, u, 0.4, 12.0, 1e-10));
            putd(p + ".phi1v", gliosim::phi1v(7.5, a, x, 1e-10));
            putd(p + ".expmv", gliosim::expmv(7.5, a, x, 1e-10));
        }
    }
    puti("stencil.count", idx);
}

// select_params over the test_expact.cpp:53-66 grid plus the BASELINE configs' norms.
void select_kats() {
    std::vector<double> norms = {0.0, 1e-6, 0.4, 1.0, 3.0, 6.0, 25.0, 4000.0, 1.2556, 3.1369, 56.637, 21.0725, 84.955,
                                 1e5, 1e9};
    std::vector<double> tols = {1e-6, 1e-8, 1e-10, 1e-12, 1e-13};
    std::vector<double> nn, tt;
    std::vector<int64_t> ss, mm;
    for (double n : norms)
        for (double t : tols) {
            gliosim::ActionParams p = gliosim::select_params(n, t);
            nn.push_back(n);
            tt.push_back(t);
            ss.push_back(p.s);
            mm.push_back(p.m);
        }
    putd("select.norm", nn);
    putd("select.tol", tt);
    puti("select.s", ss);
    puti("select.m", mm);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 2) {
        std::fprintf(stderr, "usage: gen_golden OUT\n");
        return 1;
    }
    g_out = std::fopen(argv[1], "wb");
    if (!g_out) return 1;
    select_kats();
    random_operator_kats("expmv_rand", 20260822, 5, 25, 0.5, 8.0, 30, 1e-10, false, false);  // test_expact.cpp:79-96
    random_operator_kats("phi1v_rand", 99172, 5, 22, 0.5, 8.0, 30, 1e-10, true, false);      // test_expact.cpp:146-175
    random_operator_kats("accept_c1", 20260822, 4, 30, 0.5, 10.0, 50, 1e-13, true, true);    // acceptance.cpp:57-86
    stencil_kats();
    std::fclose(g_out);
    return 0;
}
