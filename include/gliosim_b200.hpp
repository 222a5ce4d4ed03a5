// gliosim_b200.hpp -- C++ drop-in layer over the C-ABI (include/gliosim_b200.h).
//
// The reference gliosim library is C++ (/root/reference/proj/include/gliosim/*.hpp); this
// header gives its callers the same free functions with the same argument meaning, value
// semantics and exception types, backed by the B200 kernels:
//
//   reference                                             here (namespace gliosim_b200)
//   SparseOperator assemble_diffusion(const DiffusionField&)   StencilOperator assemble_diffusion(d)
//     (stencil.hpp:20)                                          (any type with .grid.{nx,ny,nz,h} and .d)
//   std::vector<double> expmv(t, A, b, tol, workers)           expmv(t, A, b, tol)      (expact.hpp:45-46)
//   std::vector<double> phi1v(t, A, b, tol, workers)           phi1v(t, A, b, tol)      (expact.hpp:49-50)
//   ActionParams select_params(norm, tol)                      select_params(norm, tol) (expact.hpp:42)
//   std::vector<double> step(A, u, rho, tau, tol, workers)     step(A, u, rho, tau, tol) (integrator.hpp:59-60)
//   RunResult run(cfg, d, u0, workers, sink, warn, watch)      run(cfg, d, u0, sink, warn, watch)
//                                                               (integrator.hpp:75-77)
//   write_vtk / read_vtk / write_metrics_csv (vtk.hpp:40-48)   same names (byte-identical files)
//   load_stack / load_raw_volume / resample / matter_fractions  same names (imaging.hpp:28-54); resample and
//     / write_label_volume / read_label_volume               matter_fractions run on the GPU
//   RunResult run_to_directory(cfg, d, materials, dir, ...)    run_to_directory(...) (pipeline.hpp:18-24),
//                                                               snapshots written while the GPU steps on
//   std::invalid_argument / numeric_error / data_error         same std::invalid_argument /
//                                                               gliosim_b200::numeric_error / data_error
//
// The reference's own types (SimConfig, DiffusionField, Grid) are accepted as template
// parameters, so a reference caller switches by changing the namespace and linking
// libgliosim_b200.so -- no reference header is needed to compile this file.
// `workers` arguments are accepted and ignored (the reference documents that results do
// not depend on them, sparse.hpp:27-29).
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "gliosim_b200.h"

namespace gliosim_b200 {

struct data_error : std::runtime_error {
    explicit data_error(const std::string& m) : std::runtime_error(m) {}
};
struct numeric_error : std::runtime_error {
    explicit numeric_error(const std::string& m) : std::runtime_error(m) {}
};
struct device_error : std::runtime_error {
    explicit device_error(const std::string& m) : std::runtime_error(m) {}
};

inline void check(gs_status st, const gs_ctx* ctx) {
    if (st == GS_OK) return;
    const std::string msg = gs_last_error(ctx);
    switch (st) {
        case GS_EINVAL: throw std::invalid_argument(msg);
        case GS_ENUMERIC: throw numeric_error(msg);
        case GS_EDATA: throw data_error(msg);
        default: throw device_error(msg);
    }
}

struct ActionParams {  // expact.hpp:33-37
    int s = 1;
    int m = 1;
    double tol = 1e-8;
};

struct StepMetrics {  // integrator.hpp:30-37
    int step = 0;
    double time = 0.0, total_mass = 0.0, max_density = 0.0, min_density = 0.0, radius = 0.0;
};

struct RunTimings {  // integrator.hpp:39-43
    double assemble_seconds = 0.0, step_seconds = 0.0, io_seconds = 0.0;
};

struct RunResult {  // integrator.hpp:45-49
    std::vector<StepMetrics> metrics;
    std::vector<double> u;
    RunTimings timings;
};

using SnapshotSink = std::function<void(int, double, const std::vector<double>&)>;
using RangeWarning = std::function<void(int, double, double)>;
using StepWatcher = std::function<void(const StepMetrics&)>;

// The device-resident, matrix-free form of the reference's SparseOperator for the
// diffusion stencil.  Move-only (it owns the device buffers of one grid).
class StencilOperator {
public:
    StencilOperator(int nx, int ny, int nz, double h, int device = 0) : nx_(nx), ny_(ny), nz_(nz), h_(h) {
        check(gs_create(&ctx_, nx, ny, nz, h, device), nullptr);
    }
    StencilOperator(StencilOperator&& o) noexcept { *this = std::move(o); }
    StencilOperator& operator=(StencilOperator&& o) noexcept {
        std::swap(ctx_, o.ctx_);
        nx_ = o.nx_;
        ny_ = o.ny_;
        nz_ = o.nz_;
        h_ = o.h_;
        return *this;
    }
    StencilOperator(const StencilOperator&) = delete;
    StencilOperator& operator=(const StencilOperator&) = delete;
    ~StencilOperator() {
        if (ctx_) gs_destroy(ctx_);
    }

    int64_t dim() const { return static_cast<int64_t>(nx_) * ny_ * nz_; }   // sparse.hpp:20
    double one_norm() const {                                                  // sparse.hpp:22
        double v = 0.0;
        check(gs_one_norm(ctx_, &v), ctx_);
        return v;
    }
    void apply(const std::vector<double>& x, std::vector<double>& y, int = 1) const {  // sparse.hpp:29
        if (static_cast<int64_t>(x.size()) != dim())
            throw std::invalid_argument("SparseOperator::apply: vector length " + std::to_string(x.size()) +
                                        " != dim " + std::to_string(dim()));
        y.resize(x.size());
        check(gs_apply(ctx_, x.data(), y.data()), ctx_);
    }
    std::vector<double> apply(const std::vector<double>& x, int workers = 1) const {
        std::vector<double> y;
        apply(x, y, workers);
        return y;
    }
    void set_diffusion(const std::vector<double>& d) { check(gs_set_diffusion(ctx_, d.data()), ctx_); }
    void set_labels(const std::vector<uint8_t>& l, double dw, double dg) {
        check(gs_set_labels(ctx_, l.data(), dw, dg), ctx_);
    }
    gs_ctx* ctx() const { return ctx_; }
    int nx() const { return nx_; }
    int ny() const { return ny_; }
    int nz() const { return nz_; }
    double h() const { return h_; }

private:
    gs_ctx* ctx_ = nullptr;
    int nx_ = 0, ny_ = 0, nz_ = 0;
    double h_ = 1.0;
};

// assemble_diffusion (stencil.cpp:5-43) for any DiffusionField-like type.
template <class DiffusionFieldT>
StencilOperator assemble_diffusion(const DiffusionFieldT& d, int device = 0) {
    StencilOperator op(d.grid.nx, d.grid.ny, d.grid.nz, d.grid.h, device);
    op.set_diffusion(d.d);
    return op;
}

inline ActionParams select_params(double norm_tA, double tol) {
    ActionParams p;
    p.tol = tol;
    check(gs_select_params(norm_tA, tol, &p.s, &p.m), nullptr);
    return p;
}

inline std::vector<double> expmv(double t, const StencilOperator& a, const std::vector<double>& b, double tol,
                                 int = 1) {
    if (static_cast<int64_t>(b.size()) != a.dim())
        throw std::invalid_argument("expmv: vector length does not match operator dimension");
    std::vector<double> out(b.size());
    check(gs_expmv(a.ctx(), t, b.data(), tol, out.data(), nullptr), a.ctx());
    return out;
}

inline std::vector<double> phi1v(double t, const StencilOperator& a, const std::vector<double>& b, double tol,
                                 int = 1) {
    if (static_cast<int64_t>(b.size()) != a.dim())
        throw std::invalid_argument("phi1v: vector length does not match operator dimension");
    std::vector<double> out(b.size());
    check(gs_phi1v(a.ctx(), t, b.data(), tol, out.data(), nullptr), a.ctx());
    return out;
}

// step (integrator.cpp:52-63).  Value semantics: the step runs on the context's staging
// buffer, the operator's resident state (run) is untouched, and concurrent calls on one
// operator are serialised by the context.  A length mismatch throws what the reference's
// first use of u throws: SparseOperator::apply's message (sparse.cpp:44-46).
inline std::vector<double> step(const StencilOperator& a, const std::vector<double>& u, double rho, double tau,
                                double tol, int = 1) {
    if (static_cast<int64_t>(u.size()) != a.dim())
        throw std::invalid_argument("SparseOperator::apply: vector length " + std::to_string(u.size()) + " != dim " +
                                    std::to_string(a.dim()));
    std::vector<double> out(u.size());
    check(gs_step_host(a.ctx(), u.data(), rho, tau, tol, out.data(), nullptr), a.ctx());
    return out;
}

namespace detail {

// Where snapshot nodes go: the caller's SnapshotSink (a host copy per node) and/or the
// library's asynchronous VTK writer (gs_snapshot_vtk) for run_to_directory.
struct VtkSink {
    std::string dir;
    const std::vector<uint8_t>* labels = nullptr;
};

template <class SimConfigT, class DiffusionFieldT>
RunResult run_impl(const SimConfigT& cfg, const DiffusionFieldT& d, std::vector<double> u0,
                   const SnapshotSink& snapshot, const RangeWarning& on_range, const StepWatcher& on_step,
                   const VtkSink* vtk, bool seed_from_cfg = false) {
    const int64_t n = static_cast<int64_t>(d.grid.nx) * d.grid.ny * d.grid.nz;
    const double center[3] = {cfg.seed_center[0], cfg.seed_center[1], cfg.seed_center[2]};
    // compute_metrics places points with the DiffusionField's grid (integrator.cpp:65-89)
    const double gorigin[3] = {d.grid.origin[0], d.grid.origin[1], d.grid.origin[2]};
    if (!seed_from_cfg) cfg.validate();
    if (!seed_from_cfg && static_cast<int64_t>(u0.size()) != n)
        throw std::invalid_argument("run: initial state length does not match the grid");
    if (static_cast<int64_t>(d.d.size()) != n)
        throw std::invalid_argument("run: diffusion field length does not match the grid");
    RunResult res;
    StencilOperator a = gliosim_b200::assemble_diffusion(d);
    if (seed_from_cfg) {  // seed_initial(d, cfg) (integrator.cpp:32-50), on the operator's own D mask
        u0.resize(static_cast<size_t>(n));
        check(gs_seed_initial(a.ctx(), gorigin, cfg.seed_amplitude, cfg.seed_width, center, 1, u0.data()), a.ctx());
        cfg.validate();
    }
    check(gs_set_state(a.ctx(), u0.data()), a.ctx());
    const double tau = (cfg.t_end - cfg.t0) / cfg.num_steps;
    auto time_at = [&](int k) { return k >= cfg.num_steps ? cfg.t_end : cfg.t0 + k * tau; };
    const bool sinks = snapshot || vtk;
    auto emit = [&](int k, const std::vector<double>* host) {
        const auto tic = std::chrono::steady_clock::now();
        if (snapshot) {
            if (host) {
                snapshot(k, time_at(k), *host);
            } else {
                std::vector<double> u(static_cast<size_t>(n));
                check(gs_get_state(a.ctx(), u.data()), a.ctx());
                snapshot(k, time_at(k), u);
            }
        }
        if (vtk) {
            char name[32];
            std::snprintf(name, sizeof name, "snapshot_%04d.vtk", k);
            const std::string path = vtk->dir + "/" + name;
            check(gs_snapshot_vtk(a.ctx(), path.c_str(), gorigin, vtk->labels ? vtk->labels->data() : nullptr),
                  a.ctx());
        }
        res.timings.io_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
    };
    emit(0, &u0);
    int done = 0;
    std::vector<gs_metrics> m;
    // segment ends: the snapshot nodes; every step when a StepWatcher / RangeWarning is given,
    // so they fire live after each step as in the reference's loop (integrator.cpp:128-131)
    const bool live = static_cast<bool>(on_step) || static_cast<bool>(on_range);
    while (done < cfg.num_steps) {
        int cut = cfg.num_steps;
        if (live)
            cut = done + 1;
        else if (sinks)
            for (int k = done + 1; k <= cfg.num_steps; ++k)
                if (k % cfg.snapshot_every == 0 || k == cfg.num_steps) {
                    cut = k;
                    break;
                }
        const int k = cut - done;
        m.assign(static_cast<size_t>(k) + 1, gs_metrics{});
        const auto tic = std::chrono::steady_clock::now();
        check(gs_run(a.ctx(), k, cfg.rho, tau, cfg.exp_tol, gorigin, center, cfg.front_threshold, m.data(), nullptr),
              a.ctx());
        res.timings.step_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
        for (int q = done == 0 ? 0 : 1; q <= k; ++q) {
            StepMetrics sm{done + q, time_at(done + q), m[q].total_mass, m[q].max_density, m[q].min_density,
                           m[q].radius};
            res.metrics.push_back(sm);
            if (done + q == 0) continue;
            if (on_step) on_step(sm);  // integrator.cpp:128-131
            if (on_range && (sm.min_density < -0.01 || sm.max_density > 1.01))
                on_range(sm.step, sm.min_density, sm.max_density);
        }
        done = cut;
        if (sinks && (cut % cfg.snapshot_every == 0 || cut == cfg.num_steps)) emit(cut, nullptr);
    }
    if (vtk) {
        const auto tic = std::chrono::steady_clock::now();
        check(gs_snapshot_flush(a.ctx()), a.ctx());
        res.timings.io_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
    }
    res.u.resize(static_cast<size_t>(n));
    check(gs_get_state(a.ctx(), res.u.data()), a.ctx());
    return res;
}

}  // namespace detail

// run (integrator.cpp:91-138) for SimConfig- and DiffusionField-like types: the time loop on
// the GPU (one launch sequence per snapshot segment), metrics computed on the device at every
// node, hooks fired in the reference's order.
template <class SimConfigT, class DiffusionFieldT>
RunResult run(const SimConfigT& cfg, const DiffusionFieldT& d, std::vector<double> u0, int = 1,
              const SnapshotSink& snapshot = {}, const RangeWarning& on_range = {}, const StepWatcher& on_step = {}) {
    return detail::run_impl(cfg, d, std::move(u0), snapshot, on_range, on_step, nullptr);
}

// ---- files (vtk.hpp:40-48): byte-identical to the reference's writers -------------------
namespace detail {
inline void check_free(gs_status st) { check(st, nullptr); }

template <class MaterialVolumeT>
std::vector<uint8_t> label_bytes(const MaterialVolumeT& mv) {
    std::vector<uint8_t> out(mv.labels.size());
    for (size_t v = 0; v < out.size(); ++v) out[v] = static_cast<uint8_t>(mv.labels[v]);
    return out;
}
}  // namespace detail

// write_vtk (vtk.cpp:59-91) for ScalarField- and MaterialVolume-like types.
template <class ScalarFieldT>
void write_vtk(const ScalarFieldT& u, const std::string& path) {
    const auto& g = u.grid;
    if (static_cast<int64_t>(u.values.size()) != static_cast<int64_t>(g.nx) * g.ny * g.nz)
        throw std::invalid_argument("write_vtk: field length does not match its grid");
    const double o[3] = {g.origin[0], g.origin[1], g.origin[2]};
    detail::check_free(gs_write_vtk(path.c_str(), u.values.data(), g.nx, g.ny, g.nz, g.h, o, nullptr, 0));
}

template <class ScalarFieldT, class MaterialVolumeT>
void write_vtk(const ScalarFieldT& u, const std::string& path, const MaterialVolumeT* materials) {
    if (!materials) return write_vtk(u, path);
    const auto& g = u.grid;
    if (static_cast<int64_t>(u.values.size()) != static_cast<int64_t>(g.nx) * g.ny * g.nz)
        throw std::invalid_argument("write_vtk: field length does not match its grid");
    if (materials->labels.size() != u.values.size())
        throw std::invalid_argument("write_vtk: material volume does not match the field grid");
    const std::vector<uint8_t> lab = detail::label_bytes(*materials);
    const double o[3] = {g.origin[0], g.origin[1], g.origin[2]};
    detail::check_free(gs_write_vtk(path.c_str(), u.values.data(), g.nx, g.ny, g.nz, g.h, o, lab.data(), 0));
}

// read_vtk (vtk.cpp:93-143): ScalarFieldT needs a default constructor, .grid (nx, ny, nz, h,
// origin) and .values, e.g. gliosim_b200::read_vtk<gliosim::ScalarField>(path).
template <class ScalarFieldT>
ScalarFieldT read_vtk(const std::string& path) {
    int dims[3];
    double h = 0.0, o[3];
    detail::check_free(gs_read_vtk(path.c_str(), dims, &h, o, nullptr, 0, 0));
    ScalarFieldT f;
    f.grid = decltype(f.grid)(dims[0], dims[1], dims[2], h, {o[0], o[1], o[2]});
    f.values.resize(static_cast<size_t>(dims[0]) * dims[1] * dims[2]);
    detail::check_free(gs_read_vtk(path.c_str(), dims, &h, o, f.values.data(),
                                   static_cast<int64_t>(f.values.size()), 0));
    return f;
}

// write_metrics_csv (vtk.cpp:145-157) for any range of StepMetrics-like records.
template <class SeriesT>
void write_metrics_csv(const SeriesT& series, const std::string& path) {
    std::vector<int32_t> step;
    std::vector<double> time;
    std::vector<gs_metrics> m;
    for (const auto& r : series) {
        step.push_back(r.step);
        time.push_back(r.time);
        m.push_back({r.total_mass, r.max_density, r.min_density, r.radius});
    }
    detail::check_free(gs_write_metrics_csv(path.c_str(), static_cast<int>(step.size()), step.data(), time.data(),
                                            m.data()));
}

// ---- imaging (imaging.hpp:28-54): loaders on the host, the material map on the GPU -----
// load_stack / load_raw_volume for any ImageStack-like type (width, height, num_slices,
// intensities), e.g. gliosim_b200::load_stack<gliosim::ImageStack>(paths).
template <class ImageStackT>
ImageStackT load_stack(const std::vector<std::string>& paths) {
    std::vector<const char*> cp;
    for (const auto& s : paths) cp.push_back(s.c_str());
    int w = 0, h = 0, n = 0;
    detail::check_free(gs_load_stack(cp.data(), static_cast<int>(cp.size()), &w, &h, &n, nullptr, 0));
    ImageStackT st;
    st.width = w;
    st.height = h;
    st.num_slices = n;
    st.intensities.resize(static_cast<size_t>(w) * h * n);
    detail::check_free(gs_load_stack(cp.data(), static_cast<int>(cp.size()), &w, &h, &n, st.intensities.data(),
                                     static_cast<int64_t>(st.intensities.size())));
    return st;
}

template <class ImageStackT>
ImageStackT load_raw_volume(const std::string& path) {
    int w = 0, h = 0, n = 0;
    detail::check_free(gs_load_raw_volume(path.c_str(), &w, &h, &n, nullptr, 0));
    ImageStackT st;
    st.width = w;
    st.height = h;
    st.num_slices = n;
    st.intensities.resize(static_cast<size_t>(w) * h * n);
    detail::check_free(gs_load_raw_volume(path.c_str(), &w, &h, &n, st.intensities.data(),
                                          static_cast<int64_t>(st.intensities.size())));
    return st;
}

// resample (imaging.cpp:118-141: nearest source + classify) on the GPU (K1), returning the
// caller's MaterialVolume type, e.g. resample<gliosim::MaterialVolume>(stack, grid, cfg).
template <class MaterialVolumeT, class ImageStackT, class GridT, class SimConfigT>
MaterialVolumeT resample(const ImageStackT& stack, const GridT& grid, const SimConfigT& cfg, int device = 0) {
    if (stack.num_slices < 1 || stack.width < 1 || stack.height < 1) throw data_error("resample: degenerate stack");
    StencilOperator op(grid.nx, grid.ny, grid.nz, grid.h, device);
    check(gs_set_intensity(op.ctx(), stack.intensities.data(), stack.width, stack.height, stack.num_slices,
                           cfg.threshold_air, cfg.threshold_white, cfg.threshold_gray, cfg.d_white, cfg.d_gray),
          op.ctx());
    std::vector<uint8_t> lab(static_cast<size_t>(op.dim()));
    check(gs_get_labels(op.ctx(), lab.data()), op.ctx());
    MaterialVolumeT mv(grid);
    using M = typename std::decay<decltype(mv.labels[0])>::type;
    for (size_t v = 0; v < lab.size(); ++v) mv.labels[v] = static_cast<M>(lab[v]);
    return mv;
}

// matter_fractions (imaging.cpp:155-164), counted on the GPU.
struct MatterFractions {
    double white = 0.0, gray = 0.0;
};
template <class MaterialVolumeT>
MatterFractions matter_fractions(const MaterialVolumeT& mv, int device = 0) {
    StencilOperator op(mv.grid.nx, mv.grid.ny, mv.grid.nz, mv.grid.h, device);
    op.set_labels(detail::label_bytes(mv), 0.13, 0.013);
    MatterFractions f;
    check(gs_matter_fractions(op.ctx(), &f.white, &f.gray), op.ctx());
    return f;
}

template <class MaterialVolumeT>
void write_label_volume(const MaterialVolumeT& mv, const std::string& path) {
    const std::vector<uint8_t> lab = detail::label_bytes(mv);
    detail::check_free(gs_write_label_volume(path.c_str(), lab.data(), mv.grid.nx, mv.grid.ny, mv.grid.nz));
}

template <class MaterialVolumeT, class GridT>
MaterialVolumeT read_label_volume(const std::string& path, const GridT& grid) {
    std::vector<uint8_t> lab(static_cast<size_t>(grid.nx) * grid.ny * grid.nz);
    detail::check_free(gs_read_label_volume(path.c_str(), grid.nx, grid.ny, grid.nz, lab.data()));
    MaterialVolumeT mv(grid);
    using M = typename std::decay<decltype(mv.labels[0])>::type;
    for (size_t v = 0; v < lab.size(); ++v) mv.labels[v] = static_cast<M>(lab[v]);
    return mv;
}

// run_to_directory (pipeline.cpp:30-53): seed from cfg (integrator.cpp:32-50, D-masked), run on
// the GPU, snapshot_NNNN.vtk at every snapshot node (with the material array when given) written
// by the library's writer thread while later steps run, then metrics.csv.
template <class SimConfigT, class DiffusionFieldT, class MaterialVolumeT>
RunResult run_to_directory(const SimConfigT& cfg, const DiffusionFieldT& d, const MaterialVolumeT* materials,
                           const std::string& out_dir, int = 1, const StepWatcher& on_step = {},
                           const RangeWarning& on_range = {}) {
    try {
        std::filesystem::create_directories(out_dir);
    } catch (const std::filesystem::filesystem_error& e) {
        throw data_error("cannot create output directory " + out_dir + ": " + e.what());
    }
    const int64_t n = static_cast<int64_t>(d.grid.nx) * d.grid.ny * d.grid.nz;
    std::vector<uint8_t> lab;
    if (materials) {
        if (static_cast<int64_t>(materials->labels.size()) != n)
            throw std::invalid_argument("write_vtk: material volume does not match the field grid");
        lab = detail::label_bytes(*materials);
    }
    const detail::VtkSink sink{out_dir, materials ? &lab : nullptr};
    RunResult res = detail::run_impl(cfg, d, {}, {}, on_range, on_step, &sink, true);
    const auto tic = std::chrono::steady_clock::now();
    write_metrics_csv(res.metrics, out_dir + "/metrics.csv");
    res.timings.io_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
    return res;
}

}  // namespace gliosim_b200
