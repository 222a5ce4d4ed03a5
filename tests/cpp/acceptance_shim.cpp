// acceptance_shim.cpp -- TEST: the reference's own acceptance program (proj/tests/acceptance.cpp,
// compiled UNMODIFIED from /root/reference) linked against the GPU drop-in instead of the
// reference's exponential integrator.
//
// oracle/Makefile target `accept` links acceptance.cpp with every reference object EXCEPT
// expact.o and integrator.o; this file defines the functions those two provide
// (expact.hpp:42-50, integrator.hpp:51-77) on top of the C ABI / C++ drop-in, so every call
// the acceptance criteria make -- directly or through pipeline.cpp (run_to_directory,
// wave_speed_experiment) -- runs on the B200:
//   * run(cfg, DiffusionField, ...)      -> gliosim_b200::run (matrix-free stencil, hooks)
//   * step / expmv / phi1v(SparseOperator) -> the device CSR path (gs_create_csr), the
//     operator uploaded once per distinct SparseOperator
//   * select_params, seed_initial, compute_metrics -> gs_select_params, gs_seed_initial and
//     a 0-step gs_run (device metrics)
// Exceptions come back as the reference's types with the library's (= the reference's)
// messages.
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "gliosim/errors.hpp"
#include "gliosim/expact.hpp"
#include "gliosim/integrator.hpp"
#include "gliosim_b200.hpp"

namespace {

// gliosim_b200 exceptions -> the reference's types (errors.hpp)
template <class F>
auto translate(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const gliosim_b200::numeric_error& e) {
        throw gliosim::numeric_error(e.what());
    } catch (const gliosim_b200::data_error& e) {
        throw gliosim::data_error(e.what());
    }
}

void check(gs_status st, const gs_ctx* c) { gliosim_b200::check(st, c); }

// One device context per distinct CSR operator (same arrays and sizes), created on first use.
struct CsrCtx {
    gs_ctx* ctx = nullptr;
    ~CsrCtx() {
        if (ctx) gs_destroy(ctx);
    }
};
std::mutex g_mu;
std::map<std::tuple<const void*, const void*, std::int64_t, std::size_t>, std::unique_ptr<CsrCtx>> g_csr;

gs_ctx* csr_ctx(const gliosim::SparseOperator& a) {
    const auto& offs = a.row_offsets();
    const auto& cols = a.column_indices();
    const auto& vals = a.coefficients();
    const auto key = std::make_tuple(static_cast<const void*>(vals.data()), static_cast<const void*>(offs.data()),
                                     a.dim(), vals.size());
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_csr.find(key);
    if (it != g_csr.end()) return it->second->ctx;
    auto c = std::make_unique<CsrCtx>();
    check(gs_create_csr(&c->ctx, a.dim(), offs.data(), cols.data(), vals.data(), 0), nullptr);
    gs_ctx* ctx = c->ctx;
    g_csr[key] = std::move(c);
    return ctx;
}

gs_ctx* grid_ctx(const gliosim::Grid& g) {
    gs_ctx* c = nullptr;
    check(gs_create(&c, g.nx, g.ny, g.nz, g.h, 0), nullptr);
    return c;
}

}  // namespace

namespace gliosim {

ActionParams select_params(double norm_tA, double tol) {
    ActionParams p;
    p.tol = tol;
    const gs_status st = gs_select_params(norm_tA, tol, &p.s, &p.m);
    if (st == GS_EINVAL) throw std::invalid_argument(gs_last_error(nullptr));
    if (st == GS_ENUMERIC) throw numeric_error(gs_last_error(nullptr));
    return p;
}

std::vector<double> expmv(double t, const SparseOperator& a, const std::vector<double>& b, double tol, int) {
    if (b.size() != static_cast<std::size_t>(a.dim()))
        throw std::invalid_argument("expmv: vector length does not match operator dimension");
    return translate([&] {
        gs_ctx* c = csr_ctx(a);
        std::vector<double> out(b.size());
        check(gs_expmv(c, t, b.data(), tol, out.data(), nullptr), c);
        return out;
    });
}

std::vector<double> phi1v(double t, const SparseOperator& a, const std::vector<double>& b, double tol, int) {
    if (b.size() != static_cast<std::size_t>(a.dim()))
        throw std::invalid_argument("phi1v: vector length does not match operator dimension");
    return translate([&] {
        gs_ctx* c = csr_ctx(a);
        std::vector<double> out(b.size());
        check(gs_phi1v(c, t, b.data(), tol, out.data(), nullptr), c);
        return out;
    });
}

std::vector<double> step(const SparseOperator& a, const std::vector<double>& u, double rho, double tau, double tol,
                         int) {
    if (static_cast<std::int64_t>(u.size()) != a.dim())
        throw std::invalid_argument("SparseOperator::apply: vector length " + std::to_string(u.size()) + " != dim " +
                                    std::to_string(a.dim()));
    return translate([&] {
        gs_ctx* c = csr_ctx(a);
        std::vector<double> out(u.size());
        check(gs_step_host(c, u.data(), rho, tau, tol, out.data(), nullptr), c);
        return out;
    });
}

namespace {
std::vector<double> seed(const Grid& g, const SimConfig& cfg, const DiffusionField* d) {
    return translate([&] {
        gs_ctx* c = grid_ctx(g);
        std::unique_ptr<gs_ctx, void (*)(gs_ctx*)> hold(c, gs_destroy);
        if (d) check(gs_set_diffusion(c, d->d.data()), c);
        const double origin[3] = {g.origin[0], g.origin[1], g.origin[2]};
        const double center[3] = {cfg.seed_center[0], cfg.seed_center[1], cfg.seed_center[2]};
        std::vector<double> u(static_cast<std::size_t>(g.num_points()));
        check(gs_seed_initial(c, origin, cfg.seed_amplitude, cfg.seed_width, center, d ? 1 : 0, u.data()), c);
        return u;
    });
}
}  // namespace

std::vector<double> seed_initial(const Grid& grid, const SimConfig& cfg) {
    if (!grid.contains(cfg.seed_center)) throw data_error("seed center lies outside the computational domain");
    return seed(grid, cfg, nullptr);
}

std::vector<double> seed_initial(const DiffusionField& d, const SimConfig& cfg) {
    if (!d.grid.contains(cfg.seed_center)) throw data_error("seed center lies outside the computational domain");
    return seed(d.grid, cfg, &d);
}

StepMetrics compute_metrics(int step, double time, const std::vector<double>& u, const Grid& grid,
                            const SimConfig& cfg) {
    return translate([&] {
        gs_ctx* c = grid_ctx(grid);
        std::unique_ptr<gs_ctx, void (*)(gs_ctx*)> hold(c, gs_destroy);
        check(gs_set_diffusion(c, std::vector<double>(u.size(), 0.0).data()), c);
        check(gs_set_state(c, u.data()), c);
        const double origin[3] = {grid.origin[0], grid.origin[1], grid.origin[2]};
        const double center[3] = {cfg.seed_center[0], cfg.seed_center[1], cfg.seed_center[2]};
        gs_metrics m{};
        check(gs_run(c, 0, cfg.rho, 1.0, cfg.exp_tol, origin, center, cfg.front_threshold, &m, nullptr), c);
        StepMetrics r;
        r.step = step;
        r.time = time;
        r.total_mass = m.total_mass;
        r.max_density = m.max_density;
        r.min_density = m.min_density;
        r.radius = m.radius;
        return r;
    });
}

RunResult run(const SimConfig& cfg, const DiffusionField& d, std::vector<double> u0, int workers,
              const SnapshotSink& snapshot, const RangeWarning& on_range, const StepWatcher& on_step) {
    return translate([&] {
        gliosim_b200::StepWatcher watch;
        if (on_step)
            watch = [&](const gliosim_b200::StepMetrics& m) {
                StepMetrics r{m.step, m.time, m.total_mass, m.max_density, m.min_density, m.radius};
                on_step(r);
            };
        const gliosim_b200::RunResult g =
            gliosim_b200::run(cfg, d, std::move(u0), workers, snapshot, on_range, watch);
        RunResult r;
        r.u = g.u;
        r.timings.assemble_seconds = g.timings.assemble_seconds;
        r.timings.step_seconds = g.timings.step_seconds;
        r.timings.io_seconds = g.timings.io_seconds;
        for (const auto& m : g.metrics)
            r.metrics.push_back(StepMetrics{m.step, m.time, m.total_mass, m.max_density, m.min_density, m.radius});
        return r;
    });
}

}  // namespace gliosim
