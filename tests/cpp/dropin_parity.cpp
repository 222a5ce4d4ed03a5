// dropin_parity.cpp -- TEST: the C++ drop-in (include/gliosim_b200.hpp) against the UNMODIFIED
// reference library, called the way a reference user calls it.  Built in the build container
// (needs /root/reference headers) by oracle/Makefile target `dropin`; the binary travels to the
// GPU box and is run by tests/test_gpu_parity.py::test_cpp_dropin_parity.
//
// Same SimConfig / DiffusionField / u0 objects go to gliosim::run (reference, CPU) and to
// gliosim_b200::run (GPU); the final state must agree to a relative L2 of 1e-8 and the
// order-free metrics (max, min, radius) to 1e-12; step() / phi1v() / expmv() / apply() too.
// With the reference's sequential sums reproduced on the device (gs_seqsum.cuh) the states are
// in fact bit-identical, and that is gated as well.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "gliosim/config.hpp"
#include "gliosim/expact.hpp"
#include "gliosim/fields.hpp"
#include "gliosim/imaging.hpp"
#include "gliosim/integrator.hpp"
#include "gliosim/pipeline.hpp"
#include "gliosim/stencil.hpp"
#include "gliosim/vtk.hpp"
#include "gliosim_b200.hpp"
#include "oracles.hpp"  // the reference's test oracles (dense expm), proj/tests

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1.0));
}

static std::string slurp(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

int main() {
    gliosim::SimConfig cfg;
    cfg.nx = 24;
    cfg.ny = 20;
    cfg.nz = 16;
    cfg.h = 200.0 / 23.0;
    cfg.num_steps = 12;
    cfg.t_end = cfg.t0 + 12 * 33.5;
    cfg.snapshot_every = 5;
    cfg.seed_center = {100.0, 80.0, 70.0};
    cfg.seed_amplitude = 1.0;
    cfg.seed_width = 0.01;
    gliosim::DiffusionField d(cfg.grid());
    for (int k = 0; k < cfg.nz; ++k)
        for (int j = 0; j < cfg.ny; ++j)
            for (int i = 0; i < cfg.nx; ++i) {
                const double r = std::hypot(i - 12.0, j - 10.0);
                d.d[static_cast<size_t>(i + cfg.nx * (j + cfg.ny * k))] =
                    r < 6 ? cfg.d_white : (r < 9 ? cfg.d_gray : 0.0);
            }
    const std::vector<double> u0 = gliosim::seed_initial(d, cfg);
    int fails = 0;
    auto gate = [&](bool ok, const char* what, double v) {
        std::printf("[%s] %s %.3e\n", ok ? "PASS" : "FAIL", what, v);
        fails += !ok;
    };

    // run (integrator.hpp:75-77) with hooks
    std::vector<int> snaps_ref, snaps_gpu, steps_gpu;
    const gliosim::RunResult ref =
        gliosim::run(cfg, d, u0, 1, [&](int n, double, const std::vector<double>&) { snaps_ref.push_back(n); });
    const gliosim_b200::RunResult gpu = gliosim_b200::run(
        cfg, d, u0, 1, [&](int n, double, const std::vector<double>&) { snaps_gpu.push_back(n); }, {},
        [&](const gliosim_b200::StepMetrics& m) { steps_gpu.push_back(m.step); });
    gate(rel_l2(gpu.u, ref.u) <= 1e-8, "run: final u rel L2", rel_l2(gpu.u, ref.u));
    gate(gpu.u == ref.u, "run: final u bitwise", 0.0);
    gate(snaps_ref == snaps_gpu, "run: snapshot cadence", 0.0);
    gate(static_cast<int>(steps_gpu.size()) == cfg.num_steps, "run: step watcher calls", 0.0);
    double worst = 0.0;
    for (size_t q = 0; q < ref.metrics.size(); ++q) {
        worst = std::fmax(worst, std::fabs(gpu.metrics[q].max_density - ref.metrics[q].max_density));
        worst = std::fmax(worst, std::fabs(gpu.metrics[q].radius - ref.metrics[q].radius) / 200.0);
        worst = std::fmax(worst, std::fabs(gpu.metrics[q].total_mass / ref.metrics[q].total_mass - 1.0));
    }
    gate(worst <= 1e-12 && gpu.metrics.size() == ref.metrics.size(), "run: metrics", worst);

    // step / phi1v / expmv / apply / one_norm
    const gliosim::SparseOperator a = gliosim::assemble_diffusion(d);
    gliosim_b200::StencilOperator ga = gliosim_b200::assemble_diffusion(d);
    gate(ga.one_norm() == a.one_norm(), "one_norm bitwise", ga.one_norm());
    gate(ga.apply(u0) == a.apply(u0), "apply bitwise", 0.0);
    const auto s_ref = gliosim::step(a, u0, cfg.rho, cfg.tau(), cfg.exp_tol);
    const auto s_gpu = gliosim_b200::step(ga, u0, cfg.rho, cfg.tau(), cfg.exp_tol);
    gate(rel_l2(s_gpu, s_ref) <= 1e-10, "step rel L2", rel_l2(s_gpu, s_ref));
    gate(s_gpu == s_ref, "step bitwise", 0.0);
    const auto p_ref = gliosim::phi1v(40.0, a, u0, 1e-10);
    const auto p_gpu = gliosim_b200::phi1v(40.0, ga, u0, 1e-10);
    gate(rel_l2(p_gpu, p_ref) <= 1e-12, "phi1v rel L2", rel_l2(p_gpu, p_ref));
    gate(p_gpu == p_ref, "phi1v bitwise", 0.0);
    const auto e_ref = gliosim::expmv(40.0, a, u0, 1e-10);
    const auto e_gpu = gliosim_b200::expmv(40.0, ga, u0, 1e-10);
    gate(e_gpu == e_ref, "expmv bitwise", rel_l2(e_gpu, e_ref));
    const auto sp = gliosim_b200::select_params(21.0725, 1e-8);
    const auto sr = gliosim::select_params(21.0725, 1e-8);
    gate(sp.s == sr.s && sp.m == sr.m, "select_params", sp.m);
    // error behaviour: same exception types
    bool threw = false;
    try {
        gliosim_b200::phi1v(1.0, ga, std::vector<double>(3, 1.0), 1e-10);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    gate(threw, "phi1v length mismatch -> std::invalid_argument", 0.0);
    // step with a wrong length: the reference throws from SparseOperator::apply (sparse.cpp:44-46)
    std::string msg_ref, msg_gpu;
    try {
        gliosim::step(a, std::vector<double>(5, 0.5), cfg.rho, cfg.tau(), cfg.exp_tol);
    } catch (const std::invalid_argument& e) {
        msg_ref = e.what();
    }
    try {
        gliosim_b200::step(ga, std::vector<double>(5, 0.5), cfg.rho, cfg.tau(), cfg.exp_tol);
    } catch (const std::invalid_argument& e) {
        msg_gpu = e.what();
    }
    std::printf("  step length mismatch: reference \"%s\", drop-in \"%s\"\n", msg_ref.c_str(), msg_gpu.c_str());
    gate(!msg_ref.empty() && msg_ref == msg_gpu, "step length mismatch: same exception and message", 0.0);
    // the reference's operators are shareable read-only: step() from two threads on one operator
    {
        std::vector<std::vector<double>> ins, outs(6), serial;
        for (int k = 0; k < 6; ++k) {
            std::vector<double> v = u0;
            for (size_t i = 0; i < v.size(); ++i) v[i] = std::fmod(v[i] + 0.37 * k + 1e-3 * static_cast<double>(i % 97), 1.0);
            ins.push_back(v);
            serial.push_back(gliosim::step(a, v, cfg.rho, cfg.tau(), cfg.exp_tol));
        }
        auto work = [&](int first) {
            for (int r = 0; r < 3; ++r)
                for (int k = first; k < 6; k += 2) outs[k] = gliosim_b200::step(ga, ins[k], cfg.rho, cfg.tau(), cfg.exp_tol);
        };
        std::thread t0(work, 0), t1(work, 1);
        t0.join();
        t1.join();
        gate(outs == serial, "step from two threads on one operator == the reference's serial steps", 0.0);
    }

    // The property of test_integrator.cpp:122-144 on the drop-in: with no reaction, ten
    // exponential-Euler steps over [0, 500] equal one exponential action over the span --
    // against the drop-in's expmv and the dense matrix exponential, 1e-7 (the unit test's bar).
    {
        gliosim::SimConfig c2;
        c2.rho = 0.0;
        c2.nx = c2.ny = c2.nz = 6;
        c2.h = 200.0 / 5.0;
        c2.t0 = 0.0;
        c2.t_end = 500.0;
        c2.num_steps = 10;
        c2.seed_center = {100.0, 100.0, 100.0};
        c2.seed_amplitude = 0.8;
        c2.seed_width = 0.002;
        const gliosim::Grid g2 = c2.grid();
        const gliosim::DiffusionField d2(g2, 0.13);
        const std::vector<double> v0 = gliosim::seed_initial(g2, c2);
        const gliosim_b200::RunResult r2 = gliosim_b200::run(c2, d2, v0);
        gliosim_b200::StencilOperator a2 = gliosim_b200::assemble_diffusion(d2);
        const std::vector<double> one = gliosim_b200::expmv(500.0, a2, v0, 1e-10);
        const double e1 = oracles::rel_err_inf(r2.u, one);
        const gliosim::SparseOperator ar = gliosim::assemble_diffusion(d2);
        const oracles::Dense e = oracles::expm(oracles::scale(oracles::dense_from_sparse(ar), 500.0));
        const double e2 = oracles::rel_err_inf(r2.u, oracles::apply(e, v0));
        gate(e1 <= 1e-7, "10 steps (rho = 0) == one expmv over the span (test_integrator.cpp:122-144)", e1);
        gate(e2 <= 1e-7, "10 steps (rho = 0) == dense expm over the span", e2);
    }

    // run_to_directory (pipeline.hpp:18-24) with labels: the same files, read back by the
    // reference's own reader; the GPU's files re-written by the reference's writer are
    // byte-identical (formatting parity), and the states agree with the reference run.
    gliosim::MaterialVolume mv(cfg.grid());
    for (size_t v = 0; v < mv.labels.size(); ++v)
        mv.labels[v] = d.d[v] == cfg.d_white ? gliosim::Material::WhiteMatter
                       : d.d[v] == cfg.d_gray ? gliosim::Material::GrayMatter : gliosim::Material::Air;
    const std::string tmp = std::filesystem::temp_directory_path().string();
    const std::string dir_ref = tmp + "/gs_dropin_ref", dir_gpu = tmp + "/gs_dropin_gpu";
    std::filesystem::remove_all(dir_ref);
    std::filesystem::remove_all(dir_gpu);
    const gliosim::RunResult rr = gliosim::run_to_directory(cfg, d, &mv, dir_ref);
    int gpu_steps = 0;
    const gliosim_b200::RunResult rg =
        gliosim_b200::run_to_directory(cfg, d, &mv, dir_gpu, 1, [&](const gliosim_b200::StepMetrics&) { ++gpu_steps; });
    gate(gpu_steps == cfg.num_steps, "run_to_directory: step watcher calls", gpu_steps);
    bool files_ok = true, bytes_ok = true;
    double worst_snap = 0.0;
    for (int k = 0; k <= cfg.num_steps; ++k) {
        char name[32];
        std::snprintf(name, sizeof name, "/snapshot_%04d.vtk", k);
        const bool want = k % cfg.snapshot_every == 0 || k == cfg.num_steps;
        const bool a_has = std::filesystem::exists(dir_ref + name), b_has = std::filesystem::exists(dir_gpu + name);
        files_ok = files_ok && a_has == want && b_has == want;
        if (!want || !a_has || !b_has) continue;
        const gliosim::ScalarField fa = gliosim::read_vtk(dir_ref + name);
        const gliosim::ScalarField fb = gliosim::read_vtk(dir_gpu + name);
        worst_snap = std::fmax(worst_snap, rel_l2(fb.values, fa.values));
        gliosim::write_vtk(fb, dir_gpu + "/rewrite.vtk", &mv);
        bytes_ok = bytes_ok && slurp(dir_gpu + "/rewrite.vtk") == slurp(dir_gpu + name);
        const auto fc = gliosim_b200::read_vtk<gliosim::ScalarField>(dir_gpu + name);
        bytes_ok = bytes_ok && fc.values == fb.values && fc.grid.h == fb.grid.h;
    }
    gate(files_ok, "run_to_directory: snapshot files at the reference's nodes", 0.0);
    gate(bytes_ok, "run_to_directory: snapshot bytes == reference write_vtk of the same state", 0.0);
    gate(worst_snap <= 1e-8, "run_to_directory: snapshots vs reference rel L2", worst_snap);
    gate(rg.u == gliosim::read_vtk(dir_gpu + "/snapshot_0012.vtk").values, "run_to_directory: last file == u", 0.0);
    std::vector<gliosim::StepMetrics> gm;
    for (const auto& m : rg.metrics) gm.push_back({m.step, m.time, m.total_mass, m.max_density, m.min_density, m.radius});
    gliosim::write_metrics_csv(gm, dir_gpu + "/metrics_ref.csv");
    gate(slurp(dir_gpu + "/metrics_ref.csv") == slurp(dir_gpu + "/metrics.csv"), "metrics.csv bytes", 0.0);
    gate(rr.metrics.size() == rg.metrics.size(), "run_to_directory: metrics rows", 0.0);
    std::filesystem::remove_all(dir_ref);
    std::filesystem::remove_all(dir_gpu);

    // imaging: PGM stack -> resample on the GPU, label files, matter fractions
    {
        const int W = 53, H = 41, S = 7;
        gliosim::ImageStack st;
        st.width = W;
        st.height = H;
        st.num_slices = S;
        st.intensities.resize(static_cast<size_t>(W) * H * S);
        uint64_t x = 0x9e3779b97f4a7c15ull;
        for (auto& b : st.intensities) {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            const int r = static_cast<int>(x % 100);
            b = static_cast<uint8_t>(r < 10 ? 0 : r < 60 ? 150 + r : r < 90 ? 232 + r % 8 : 250);
        }
        std::vector<std::string> paths;
        for (int z = 0; z < S; ++z) {
            const std::string p = tmp + "/gs_dropin_slice_" + std::to_string(z) + ".pgm";
            std::ofstream o(p, std::ios::binary);
            o << "P5\n# dropin\n" << W << ' ' << H << "\n255\n";
            o.write(reinterpret_cast<const char*>(st.intensities.data()) + static_cast<size_t>(z) * W * H, W * H);
            paths.push_back(p);
        }
        const gliosim::ImageStack a = gliosim::load_stack(paths);
        const auto b = gliosim_b200::load_stack<gliosim::ImageStack>(paths);
        gate(a.intensities == b.intensities && a.width == b.width && a.num_slices == b.num_slices,
             "load_stack bytes", 0.0);
        const gliosim::Grid g(40, 36, 20, 2.0);
        const gliosim::MaterialVolume mr = gliosim::resample(a, g, cfg);
        const auto mg = gliosim_b200::resample<gliosim::MaterialVolume>(b, g, cfg);
        gate(mr.labels == mg.labels, "resample (GPU) labels exact", 0.0);
        const auto fr = gliosim::matter_fractions(mr);
        const auto fg = gliosim_b200::matter_fractions(mg);
        gate(fr.white == fg.white && fr.gray == fg.gray, "matter_fractions exact", fg.white);
        gliosim_b200::write_label_volume(mg, tmp + "/gs_dropin_labels.raw");
        gate(gliosim::read_label_volume(tmp + "/gs_dropin_labels.raw", g).labels == mr.labels, "label volume", 0.0);
        for (const auto& p : paths) std::filesystem::remove(p);
        std::filesystem::remove(tmp + "/gs_dropin_labels.raw");
    }

    std::printf("%s\n", fails ? "dropin parity: FAILED" : "dropin parity: all passed");
    return fails ? 1 : 0;
}
