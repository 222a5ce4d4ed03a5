/*
 * gliosim_b200.h -- C-ABI of the B200-native exponential-Euler hot path.
 *
 * Drop-in boundary for the reference gliosim library (/root/reference/proj).  Every
 * entry point names the reference interface it replaces (file:line, paths relative to
 * /root/reference/proj).  Plain pointers and sizes only; host buffers are
 * caller-owned, device memory belongs to the context.  One context = one grid operator + one
 * CUDA stream.  Calls on one context from several threads are serialised by a per-context lock
 * (the reference's operators are immutable and shareable read-only, SPEC.md), and
 * gs_last_error() returns the message of the calling thread's own last failure on that
 * context; independent contexts run concurrently.  The value-semantics calls (gs_step_host,
 * gs_phi1v, gs_expmv, gs_apply, gs_step_ensemble_host) never touch the resident state that
 * gs_set_state / gs_run / gs_get_state work on.
 *
 * Errors: every call returns a gs_status.  The codes map 1:1 onto the reference's
 * exception types (errors.hpp:10-17, std::invalid_argument); gs_last_error() returns
 * the reference's message text for the failing call.  There is no CPU fallback: a
 * missing or failing GPU returns GS_ECUDA.
 */
#ifndef GLIOSIM_B200_H
#define GLIOSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gs_status {
    GS_OK = 0,
    GS_EINVAL = 1,   /* std::invalid_argument */
    GS_ENUMERIC = 2, /* gliosim::numeric_error */
    GS_EDATA = 3,    /* gliosim::data_error */
    GS_ECUDA = 4     /* device / driver failure (no reference analogue) */
} gs_status;

#define GS_MAX_LOGGED_STAGES 256

/* What one exponential-Euler step (or phi1v / expmv) did.  The reference exposes none
 * of this; it is the parity log ((s,m) and terms-per-stage must match). */
typedef struct gs_step_info {
    int32_t s, m;            /* select_params result (expact.cpp:29-61) */
    int32_t branch;          /* 0 Taylor, 1 t == 0, 2 ||b||_1 == 0, 3 small-norm (expact.cpp:108-122) */
    int32_t reruns;          /* two-term sweeps re-run with exact maxima (a bounded test was unsettled) */
    int64_t total_terms;     /* Taylor terms = operator applications inside expmv */
    int32_t terms[GS_MAX_LOGGED_STAGES]; /* terms used per stage (expact.cpp:81-95) */
    double bnorm;            /* ||b||_1 (expact.cpp:110), device tree-reduced */
    double anorm;            /* ||A||_1 (sparse.cpp:36-40), exact */
    double coln;             /* bordered column sum sum|b_i/gamma| (sparse.cpp:36-38 on the bordered CSR) */
    double gamma;            /* bnorm / anorm (expact.cpp:126) */
    double norm_tA;          /* |t| * ||A_bordered||_1 fed to select_params */
} gs_step_info;

/* StepMetrics (integrator.hpp:30-37) minus step/time, which the caller knows. */
typedef struct gs_metrics {
    double total_mass, max_density, min_density, radius;
} gs_metrics;

typedef struct gs_ctx gs_ctx;

/* ---- context: one regular grid (Grid, grid.hpp:14-51) ------------------------------ */
/* Replaces the SparseOperator that assemble_diffusion (stencil.hpp:20, stencil.cpp:5-43)
 * builds: the operator stays matrix-free on the device.  Validation and messages follow
 * Grid's constructor (grid.hpp:24-29). */
gs_status gs_create(gs_ctx** out, int nx, int ny, int nz, double h, int device);
void gs_destroy(gs_ctx* ctx);
/* Message of the last failing call on ctx; with ctx == NULL, of the last failing call that
 * takes no context (gs_create, gs_select_params, the file functions) on this thread. */
const char* gs_last_error(const gs_ctx* ctx);
/* Number of voxels nx*ny*nz (Grid::num_points, grid.hpp:31-33). */
int64_t gs_num_points(const gs_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for callers that time or order work on it. */
void* gs_stream(gs_ctx* ctx);

/* A generic sparse operator: SparseOperator(dim, row_offsets, column_indices, coefficients)
 * (sparse.hpp:13-38), validated with the reference's rules and messages (sparse.cpp:14-35):
 * offs has dim+1 entries, offs[0] == 0, columns sorted and unique per row.  Every call below
 * that takes the operator (apply, one_norm, expmv, phi1v, step, run) then applies this matrix
 * on the GPU -- the path the reference's random-operator tests use (test_expact.cpp:79-239). */
gs_status gs_create_csr(gs_ctx** out, int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals,
                        int device);

/* ---- material map (K1) ------------------------------------------------------------ */
/* resample + classify (imaging.cpp:65-72, 118-141) on the device from a uint8 stack
 * (x-fastest, x + y*w + z*w*hgt, imaging.hpp:21-25), then the D table of
 * diffusion_from_materials (imaging.cpp:143-153).  Thresholds as SimConfig
 * (config.hpp:40-43). */
gs_status gs_set_intensity(gs_ctx* ctx, const uint8_t* stack, int w, int hgt, int slices, int t_air,
                           int t_white, int t_gray, double d_white, double d_gray);
/* MaterialVolume labels (0 Air, 1 White, 2 Gray, 3 Skull; fields.hpp:13-18) ->
 * diffusion_from_materials (imaging.cpp:143-153). */
gs_status gs_set_labels(gs_ctx* ctx, const uint8_t* labels, double d_white, double d_gray);
/* Arbitrary DiffusionField (fields.hpp:51-60) for assemble_diffusion (stencil.cpp:5-43). */
gs_status gs_set_diffusion(gs_ctx* ctx, const double* d);
/* Copy back the device material labels (valid after gs_set_intensity / gs_set_labels). */
gs_status gs_get_labels(gs_ctx* ctx, uint8_t* labels);
/* Copy back the per-voxel D(x) the operator uses. */
gs_status gs_get_diffusion(gs_ctx* ctx, double* d);

/* ---- operator ---------------------------------------------------------------------- */
/* SparseOperator::one_norm (sparse.hpp:22, sparse.cpp:36-40): exact max column sum. */
gs_status gs_one_norm(gs_ctx* ctx, double* out);
/* SparseOperator::apply (sparse.hpp:29, sparse.cpp:43-76): y = A x, host buffers. */
gs_status gs_apply(gs_ctx* ctx, const double* x, double* y);

/* ---- state ------------------------------------------------------------------------- */
gs_status gs_set_state(gs_ctx* ctx, const double* u);
gs_status gs_get_state(gs_ctx* ctx, double* u);
/* Device pointer of the resident state u (N doubles), for zero-copy callers. */
double* gs_state_device_ptr(gs_ctx* ctx);

/* ---- exponential action / integrator ------------------------------------------------ */
/* select_params (expact.hpp:42, expact.cpp:29-61). */
gs_status gs_select_params(double norm_tA, double tol, int* s, int* m);
/* expmv (expact.hpp:45-46, expact.cpp:63-99) with A = this grid's operator. */
gs_status gs_expmv(gs_ctx* ctx, double t, const double* b, double tol, double* out, gs_step_info* info);
/* phi1v (expact.hpp:49-50, expact.cpp:101-153). */
gs_status gs_phi1v(gs_ctx* ctx, double t, const double* b, double tol, double* out, gs_step_info* info);
/* step (integrator.hpp:59-60, integrator.cpp:52-63) on the RESIDENT state: u <- step(A, u). */
gs_status gs_step(gs_ctx* ctx, double rho, double tau, double tol, gs_step_info* info);
/* step with host vectors, value semantics as the reference (u in, out returned); runs on a
 * staging buffer, leaving the resident state untouched. */
gs_status gs_step_host(gs_ctx* ctx, const double* u, double rho, double tau, double tol, double* out,
                       gs_step_info* info);
/* The time loop of run (integrator.cpp:91-138) on the resident state: n_steps steps,
 * compute_metrics (integrator.cpp:65-89) at every node.  metrics: n_steps+1 records
 * (node 0 = the state on entry) or NULL; infos: n_steps records or NULL.  One device
 * launch for the whole loop. */
gs_status gs_run(gs_ctx* ctx, int n_steps, double rho, double tau, double tol, const double origin[3],
                 const double seed_center[3], double front_threshold, gs_metrics* metrics,
                 gs_step_info* infos);
/* An ensemble of independent runs (BASELINE C5; run() of integrator.cpp:91-138 per member):
 * member i is context ctxs[i] (its own operator and resident state) with rho = rhos[i],
 * origin = origins[3i..], seed centre = centers[3i..]; every member advances n_steps steps
 * with the same tau and tol.  metrics: n_members * (n_steps+1) records (member-major) or
 * NULL; infos: n_members * n_steps records or NULL.  All members live on one device.  The
 * members' steps are batched: one launch per kernel of the step serves every member, and
 * the Taylor launch runs `groups` members at a time on groups of SMs (groups <= 0: the
 * default).  Members the batched path cannot take (CSR operators, shapes without TMA,
 * mixed 2-D/3-D) run one after another through gs_run.  Each member's result is that of
 * gs_run on its own context, up to the ulps of the per-CTA partial sums. */
gs_status gs_run_ensemble(gs_ctx* const* ctxs, int n_members, int n_steps, const double* rhos, double tau,
                          double tol, const double* origins, const double* centers, double front_threshold,
                          gs_metrics* metrics, gs_step_info* infos, int groups);
/* One step of every member with host vectors (step() of integrator.cpp:52-63 per member, value
 * semantics as gs_step_host): member i's u from u_in[i], u' into u_out[i] (each ctxs[i]'s point
 * count).  The members run batched as in gs_run_ensemble, in `chunks` consecutive groups of
 * members (<= 0: the default) whose host-to-device and device-to-host copies, on their own
 * streams, overlap the other chunks' steps; with pinned host vectors the copies are
 * asynchronous.  infos: n_members records or NULL.  The resident states are overwritten. */
gs_status gs_step_ensemble_host(gs_ctx* const* ctxs, int n_members, const double* const* u_in, double* const* u_out,
                                const double* rhos, double tau, double tol, gs_step_info* infos, int groups,
                                int chunks);

/* ---- host helpers with libm parity --------------------------------------------------- */
/* seed_initial (integrator.cpp:32-50): u = amplitude*exp(-width*|x-c|^2), zero where the
 * context's D is 0 when mask != 0.  Host libm, so u0 is bit-identical to the reference. */
gs_status gs_seed_initial(gs_ctx* ctx, const double origin[3], double amplitude, double width,
                          const double center[3], int mask, double* u);

/* ---- diagnostics ---------------------------------------------------------------------- */
/* Record a per-phase timeline (grid-barrier timestamps, ns) in subsequent launches;
 * capacity = max records per launch, 0 disables.  Tags: 1 metrics(0), 2 RHS, 3 bordered
 * column, 4 fused first-term sweep, 5 fused next-terms sweep, 6 implicit-f fix-up,
 * 7 update+metrics, 8 single-term sweep, 9 degenerate branch, 15 launch start. */
gs_status gs_set_trace(gs_ctx* ctx, int capacity);
/* Copy the last launch's records as (tag, ns) pairs; *count receives the number of records. */
gs_status gs_get_trace(gs_ctx* ctx, uint64_t* pairs, int capacity, int* count);
/* Per-kernel device time with CUDA events on the context's stream around every launch
 * of the sequence (enable != 0).  gs_get_kernel_times returns, for the last gs_run /
 * gs_step / gs_phi1v / gs_expmv call, total milliseconds and launch counts of:
 * [0] prep (RHS), [1] border, [2] taylor (the Taylor-term kernel), [3] update. */
gs_status gs_set_kernel_timing(gs_ctx* ctx, int enable);
gs_status gs_get_kernel_times(gs_ctx* ctx, double ms[4], int launches[4]);
/* 1 when gs_run on this context takes the small-grid path: one thread-block cluster runs
 * every step with the state in distributed shared memory (grids up to 40 K voxels;
 * GS_NO_CLUSTER=1 disables it).  The kernel times then report it as the Taylor kernel. */
int gs_uses_cluster(const gs_ctx* ctx);
/* 1 when the Taylor loop of this context's steps (expact.cpp:63-153) takes the 2-D path: one
 * resident CTA per 32 x 32 tile with the tile in shared memory (nz == 1, every tile on the
 * device at once; GS_NO_2D=1 disables it).  In run mode gs_uses_cluster takes precedence. */
int gs_uses_flat2d(const gs_ctx* ctx);

/* ---- snapshot and metrics files (vtk.hpp:15-45, src/vtk.cpp:59-157) ------------------- */
/* write_vtk (vtk.cpp:59-91): legacy ASCII VTK, header + one "%.17g" value per line, then,
 * when labels != NULL, "SCALARS material int 1" and one label per line.  Byte-identical to
 * the reference.  threads <= 0 picks the host's core count.  Errors: GS_EDATA "cannot open
 * <path> for writing" / "write failed: <path>". */
gs_status gs_write_vtk(const char* path, const double* u, int nx, int ny, int nz, double h, const double origin[3],
                       const uint8_t* labels, int threads);
/* read_vtk (vtk.cpp:93-143), same checks and messages.  With values == NULL only the header
 * is read (dims, h, origin); otherwise capacity >= nx*ny*nz values are filled.  A trailing
 * material array is ignored. */
gs_status gs_read_vtk(const char* path, int dims[3], double* h, double origin[3], double* values, int64_t capacity,
                      int threads);
/* write_metrics_csv (vtk.cpp:145-157): "step,time_days,total_mass,max_density,radius_mm". */
gs_status gs_write_metrics_csv(const char* path, int count, const int32_t* step, const double* time,
                               const gs_metrics* metrics);
/* The snapshot sink of run_to_directory (pipeline.cpp:39-45), asynchronous: opens path now
 * (an unwritable path fails here, as write_vtk would), copies the resident state on the
 * device, lands it in pinned host memory on a side stream and formats it on a writer
 * thread while later steps run.  labels (nx*ny*nz codes) may be NULL and are copied.  At
 * most 3 snapshots are in flight; the call blocks while all are busy, and reports the
 * error of an earlier snapshot that failed. */
gs_status gs_snapshot_vtk(gs_ctx* ctx, const char* path, const double origin[3], const uint8_t* labels);
/* Wait for every queued snapshot; returns the first failure not yet reported. */
gs_status gs_snapshot_flush(gs_ctx* ctx);

/* ---- image and label files (imaging.hpp:28-54, src/imaging.cpp:14-116, 166-190) ------ */
/* load_stack: binary PGM slices (P5, maxval 255), all the same size, stacked bottom first.
 * out == NULL returns the sizes only (all files still validated); otherwise capacity >=
 * width*height*slices bytes receive the intensities (x fastest). */
gs_status gs_load_stack(const char* const* paths, int count, int* width, int* height, int* slices, uint8_t* out,
                        int64_t capacity);
/* load_raw_volume: "nx ny nz\n" then nx*ny*nz bytes.  out == NULL returns the sizes only. */
gs_status gs_load_raw_volume(const char* path, int* width, int* height, int* slices, uint8_t* out,
                             int64_t capacity);
/* write_label_volume / read_label_volume: the raw format with Material codes 0..3. */
gs_status gs_write_label_volume(const char* path, const uint8_t* labels, int nx, int ny, int nz);
gs_status gs_read_label_volume(const char* path, int nx, int ny, int nz, uint8_t* labels);
/* matter_fractions (imaging.cpp:155-164) of the context's device labels: white and gray
 * shares of the tissue voxels.  GS_EDATA when there is no tissue. */
gs_status gs_matter_fractions(gs_ctx* ctx, double* white, double* gray);

#ifdef __cplusplus
}
#endif

#endif
