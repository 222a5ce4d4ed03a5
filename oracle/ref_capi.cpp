// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library (gliosim, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  This file
// contains no reference code: it only calls the reference's public API
// (proj/include/gliosim/*.hpp) so Python tests and bench.py can drive it with
// ctypes.  Used (a) to generate/pin golden vectors, (b) as the CPU baseline and
// the reference arm of bench.py.  Never linked into the product.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gliosim/config.hpp"
#include "gliosim/errors.hpp"
#include "gliosim/expact.hpp"
#include "gliosim/imaging.hpp"
#include "gliosim/integrator.hpp"
#include "gliosim/pipeline.hpp"
#include "gliosim/sparse.hpp"
#include "gliosim/stencil.hpp"
#include "gliosim/vtk.hpp"

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 numeric_error, 3 data_error, 4 other
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const gliosim::numeric_error& e) {
        g_err = e.what();
        return 2;
    } catch (const gliosim::data_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

gliosim::DiffusionField field(int nx, int ny, int nz, double h, const double* d) {
    gliosim::Grid g(nx, ny, nz, h);
    gliosim::DiffusionField f(g);
    std::memcpy(f.d.data(), d, sizeof(double) * f.d.size());
    return f;
}

gliosim::SparseOperator csr(int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals) {
    std::vector<int64_t> o(offs, offs + dim + 1);
    std::vector<int32_t> c(cols, cols + offs[dim]);
    std::vector<double> v(vals, vals + offs[dim]);
    return gliosim::SparseOperator(dim, std::move(o), std::move(c), std::move(v));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_classify(int intensity) { return static_cast<int>(gliosim::classify(intensity, gliosim::SimConfig{})); }

int ref_resample(const uint8_t* stack, int w, int hgt, int slices, int nx, int ny, int nz, uint8_t* labels) {
    return guard([&] {
        gliosim::ImageStack s;
        s.width = w;
        s.height = hgt;
        s.num_slices = slices;
        s.intensities.assign(stack, stack + static_cast<size_t>(w) * hgt * slices);
        gliosim::MaterialVolume mv = gliosim::resample(s, gliosim::Grid(nx, ny, nz, 1.0), gliosim::SimConfig{});
        for (size_t v = 0; v < mv.labels.size(); ++v) labels[v] = static_cast<uint8_t>(mv.labels[v]);
    });
}

int ref_diffusion_from_labels(const uint8_t* labels, int nx, int ny, int nz, double* d) {
    return guard([&] {
        gliosim::MaterialVolume mv(gliosim::Grid(nx, ny, nz, 1.0));
        for (size_t v = 0; v < mv.labels.size(); ++v) mv.labels[v] = static_cast<gliosim::Material>(labels[v]);
        gliosim::DiffusionField df = gliosim::diffusion_from_materials(mv, gliosim::SimConfig{});
        std::memcpy(d, df.d.data(), sizeof(double) * df.d.size());
    });
}

int ref_seed_initial(int nx, int ny, int nz, double h, double amplitude, double width, const double* center,
                     const double* d_mask, double* u) {
    return guard([&] {
        gliosim::SimConfig cfg;
        cfg.nx = nx;
        cfg.ny = ny;
        cfg.nz = nz;
        cfg.h = h;
        cfg.seed_amplitude = amplitude;
        cfg.seed_width = width;
        cfg.seed_center = {center[0], center[1], center[2]};
        std::vector<double> r;
        if (d_mask)
            r = gliosim::seed_initial(field(nx, ny, nz, h, d_mask), cfg);
        else
            r = gliosim::seed_initial(cfg.grid(), cfg);
        std::memcpy(u, r.data(), sizeof(double) * r.size());
    });
}

// Stencil operator built by the reference's assemble_diffusion.
int ref_stencil_apply(int nx, int ny, int nz, double h, const double* d, const double* x, double* y) {
    return guard([&] {
        gliosim::SparseOperator a = gliosim::assemble_diffusion(field(nx, ny, nz, h, d));
        std::vector<double> xv(x, x + a.dim()), yv;
        a.apply(xv, yv, 1);
        std::memcpy(y, yv.data(), sizeof(double) * yv.size());
    });
}

int ref_stencil_one_norm(int nx, int ny, int nz, double h, const double* d, double* out) {
    return guard([&] { *out = gliosim::assemble_diffusion(field(nx, ny, nz, h, d)).one_norm(); });
}

int ref_stencil_nnz(int nx, int ny, int nz, double h, const double* d, int64_t* out) {
    return guard([&] { *out = gliosim::assemble_diffusion(field(nx, ny, nz, h, d)).nnz(); });
}

int ref_select_params(double norm_tA, double tol, int* s, int* m) {
    return guard([&] {
        gliosim::ActionParams p = gliosim::select_params(norm_tA, tol);
        *s = p.s;
        *m = p.m;
    });
}

int ref_csr_apply(int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals, const double* x,
                  double* y) {
    return guard([&] {
        gliosim::SparseOperator a = csr(dim, offs, cols, vals);
        std::vector<double> xv(x, x + dim), yv;
        a.apply(xv, yv, 1);
        std::memcpy(y, yv.data(), sizeof(double) * yv.size());
    });
}

int ref_csr_one_norm(int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals, double* out) {
    return guard([&] { *out = csr(dim, offs, cols, vals).one_norm(); });
}

int ref_csr_expmv(int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals, double t,
                  const double* b, int64_t blen, double tol, double* out) {
    return guard([&] {
        std::vector<double> r = gliosim::expmv(t, csr(dim, offs, cols, vals), std::vector<double>(b, b + blen), tol);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int ref_csr_phi1v(int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals, double t,
                  const double* b, int64_t blen, double tol, double* out) {
    return guard([&] {
        std::vector<double> r = gliosim::phi1v(t, csr(dim, offs, cols, vals), std::vector<double>(b, b + blen), tol);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int ref_csr_step(int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals, const double* u,
                 double rho, double tau, double tol, double* out) {
    return guard([&] {
        std::vector<double> r =
            gliosim::step(csr(dim, offs, cols, vals), std::vector<double>(u, u + dim), rho, tau, tol);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int ref_stencil_expmv(int nx, int ny, int nz, double h, const double* d, double t, const double* b, double tol,
                      double* out) {
    return guard([&] {
        gliosim::SparseOperator a = gliosim::assemble_diffusion(field(nx, ny, nz, h, d));
        std::vector<double> r = gliosim::expmv(t, a, std::vector<double>(b, b + a.dim()), tol);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int ref_stencil_phi1v(int nx, int ny, int nz, double h, const double* d, double t, const double* b, double tol,
                      double* out) {
    return guard([&] {
        gliosim::SparseOperator a = gliosim::assemble_diffusion(field(nx, ny, nz, h, d));
        std::vector<double> r = gliosim::phi1v(t, a, std::vector<double>(b, b + a.dim()), tol);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

// n_steps exponential-Euler steps through gliosim::run (integrator.cpp:91-138).
// metrics: (n_steps+1) x 4 (total_mass, max, min, radius); step_seconds: the
// reference's own RunTimings::step_seconds (integrator.cpp:123-125).
int ref_run(int nx, int ny, int nz, double h, const double* d, const double* u0, int n_steps, double rho,
            double t0, double t_end, double tol, const double* center, double front_threshold, int workers,
            double* u_out, double* metrics, double* step_seconds) {
    return guard([&] {
        gliosim::SimConfig cfg;
        cfg.nx = nx;
        cfg.ny = ny;
        cfg.nz = nz;
        cfg.h = h;
        cfg.rho = rho;
        cfg.t0 = t0;
        cfg.t_end = t_end;
        cfg.num_steps = n_steps;
        cfg.exp_tol = tol;
        cfg.seed_center = {center[0], center[1], center[2]};
        cfg.front_threshold = front_threshold;
        const size_t n = static_cast<size_t>(nx) * ny * nz;
        gliosim::RunResult res =
            gliosim::run(cfg, field(nx, ny, nz, h, d), std::vector<double>(u0, u0 + n), workers);
        if (u_out) std::memcpy(u_out, res.u.data(), sizeof(double) * n);
        if (metrics)
            for (size_t s = 0; s < res.metrics.size(); ++s) {
                metrics[4 * s + 0] = res.metrics[s].total_mass;
                metrics[4 * s + 1] = res.metrics[s].max_density;
                metrics[4 * s + 2] = res.metrics[s].min_density;
                metrics[4 * s + 3] = res.metrics[s].radius;
            }
        if (step_seconds) *step_seconds = res.timings.step_seconds;
    });
}

// One gliosim::step on the stencil operator (integrator.cpp:52-63).
int ref_stencil_step(int nx, int ny, int nz, double h, const double* d, const double* u, double rho, double tau,
                     double tol, int workers, double* out) {
    return guard([&] {
        gliosim::SparseOperator a = gliosim::assemble_diffusion(field(nx, ny, nz, h, d));
        std::vector<double> r = gliosim::step(a, std::vector<double>(u, u + a.dim()), rho, tau, tol, workers);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

// ---- file formats (vtk.cpp, imaging.cpp, pipeline.cpp) ------------------------------
int ref_write_vtk(const char* path, const double* u, int nx, int ny, int nz, double h, const double* origin,
                  const uint8_t* labels) {
    return guard([&] {
        gliosim::Grid g(nx, ny, nz, h, {origin[0], origin[1], origin[2]});
        gliosim::ScalarField f{g, std::vector<double>(u, u + g.num_points())};
        if (labels) {
            gliosim::MaterialVolume mv(g);
            for (size_t v = 0; v < mv.labels.size(); ++v) mv.labels[v] = static_cast<gliosim::Material>(labels[v]);
            gliosim::write_vtk(f, path, &mv);
        } else {
            gliosim::write_vtk(f, path);
        }
    });
}

// values == NULL: header only
int ref_read_vtk(const char* path, int* dims, double* h, double* origin, double* values, int64_t capacity) {
    return guard([&] {
        gliosim::ScalarField f = gliosim::read_vtk(path);
        dims[0] = f.grid.nx;
        dims[1] = f.grid.ny;
        dims[2] = f.grid.nz;
        *h = f.grid.h;
        for (int a = 0; a < 3; ++a) origin[a] = f.grid.origin[a];
        if (values) {
            if (capacity < static_cast<int64_t>(f.values.size())) throw std::invalid_argument("capacity");
            std::memcpy(values, f.values.data(), sizeof(double) * f.values.size());
        }
    });
}

int ref_write_metrics_csv(const char* path, int count, const int* step, const double* time, const double* m4) {
    return guard([&] {
        std::vector<gliosim::StepMetrics> s(static_cast<size_t>(count));
        for (int i = 0; i < count; ++i) {
            s[i].step = step[i];
            s[i].time = time[i];
            s[i].total_mass = m4[4 * i + 0];
            s[i].max_density = m4[4 * i + 1];
            s[i].min_density = m4[4 * i + 2];
            s[i].radius = m4[4 * i + 3];
        }
        gliosim::write_metrics_csv(s, path);
    });
}

int ref_load_stack(const char* const* paths, int count, int* dims, uint8_t* out, int64_t capacity) {
    return guard([&] {
        gliosim::ImageStack st = gliosim::load_stack(std::vector<std::string>(paths, paths + count));
        dims[0] = st.width;
        dims[1] = st.height;
        dims[2] = st.num_slices;
        if (out) {
            if (capacity < static_cast<int64_t>(st.intensities.size())) throw std::invalid_argument("capacity");
            std::memcpy(out, st.intensities.data(), st.intensities.size());
        }
    });
}

int ref_load_raw_volume(const char* path, int* dims, uint8_t* out, int64_t capacity) {
    return guard([&] {
        gliosim::ImageStack st = gliosim::load_raw_volume(path);
        dims[0] = st.width;
        dims[1] = st.height;
        dims[2] = st.num_slices;
        if (out) {
            if (capacity < static_cast<int64_t>(st.intensities.size())) throw std::invalid_argument("capacity");
            std::memcpy(out, st.intensities.data(), st.intensities.size());
        }
    });
}

int ref_write_label_volume(const char* path, const uint8_t* labels, int nx, int ny, int nz) {
    return guard([&] {
        gliosim::MaterialVolume mv(gliosim::Grid(nx, ny, nz, 1.0));
        for (size_t v = 0; v < mv.labels.size(); ++v) mv.labels[v] = static_cast<gliosim::Material>(labels[v]);
        gliosim::write_label_volume(mv, path);
    });
}

int ref_read_label_volume(const char* path, int nx, int ny, int nz, uint8_t* labels) {
    return guard([&] {
        gliosim::MaterialVolume mv = gliosim::read_label_volume(path, gliosim::Grid(nx, ny, nz, 1.0));
        for (size_t v = 0; v < mv.labels.size(); ++v) labels[v] = static_cast<uint8_t>(mv.labels[v]);
    });
}

int ref_matter_fractions(const uint8_t* labels, int nx, int ny, int nz, double* white, double* gray) {
    return guard([&] {
        gliosim::MaterialVolume mv(gliosim::Grid(nx, ny, nz, 1.0));
        for (size_t v = 0; v < mv.labels.size(); ++v) mv.labels[v] = static_cast<gliosim::Material>(labels[v]);
        const gliosim::MatterFractions f = gliosim::matter_fractions(mv);
        *white = f.white;
        *gray = f.gray;
    });
}

// run_to_directory (pipeline.cpp:30-53) with a DiffusionField d and optional labels.
// io_seconds: the reference's RunTimings::io_seconds (snapshot + csv time).
int ref_run_to_directory(int nx, int ny, int nz, double h, const double* d, const uint8_t* labels, int n_steps,
                         int snapshot_every, double rho, double t0, double t_end, double tol, const double* center,
                         double amplitude, double width, const char* out_dir, double* u_out, double* step_seconds,
                         double* io_seconds) {
    return guard([&] {
        gliosim::SimConfig cfg;
        cfg.nx = nx;
        cfg.ny = ny;
        cfg.nz = nz;
        cfg.h = h;
        cfg.rho = rho;
        cfg.t0 = t0;
        cfg.t_end = t_end;
        cfg.num_steps = n_steps;
        cfg.snapshot_every = snapshot_every;
        cfg.exp_tol = tol;
        cfg.seed_center = {center[0], center[1], center[2]};
        cfg.seed_amplitude = amplitude;
        cfg.seed_width = width;
        gliosim::DiffusionField f = field(nx, ny, nz, h, d);
        gliosim::MaterialVolume mv(f.grid);
        if (labels)
            for (size_t v = 0; v < mv.labels.size(); ++v) mv.labels[v] = static_cast<gliosim::Material>(labels[v]);
        gliosim::RunResult r = gliosim::run_to_directory(cfg, f, labels ? &mv : nullptr, out_dir);
        if (u_out) std::memcpy(u_out, r.u.data(), sizeof(double) * r.u.size());
        if (step_seconds) *step_seconds = r.timings.step_seconds;
        if (io_seconds) *io_seconds = r.timings.io_seconds;
    });
}

}  // extern "C"
