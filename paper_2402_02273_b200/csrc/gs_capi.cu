// gs_capi.cu -- host side of the C-ABI (include/gliosim_b200.h).
//
// Owns the device state of one grid operator and drives the kernels of gs_kernels.cu.
// The host does exactly the libm-dependent scalar work the reference does with glibc
// (r_m of select_params, expact.cpp:47-48; the Gaussian seed, integrator.cpp:40-41) so
// those values are bit-identical; everything per-voxel runs on the GPU.  No CPU
// fallback exists: without a device every entry point returns GS_ECUDA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gliosim_b200.h"
#include "gs_io.hpp"
#include "gs_kernels.cuh"
#include "gs_vtkfmt.cuh"

namespace {

thread_local std::string g_create_error;
// the last failure on this thread and its context: gs_last_error(ctx) reads it first, so another
// thread's later failure on the same context cannot overwrite the message a caller is reading
thread_local std::string t_err;
thread_local const void* t_err_ctx = nullptr;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t alloc(size_t b) {
        if (bytes >= b && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// Asynchronous snapshot sink (gs_snapshot_vtk): a device copy of the state per slot, a
// pinned host copy landed by the side stream, and one writer thread per context.
constexpr int kSnapSlots = 3;

// Grids up to this many voxels run whole gs_run calls in one thread-block cluster.
constexpr int64_t kClusterMaxVoxels = 40000;

// Taylor terms per fused TMA sweep (2 or 3); GS_FUSE overrides it per launch.
constexpr int kDefaultFuse = 2;

// gs_run_ensemble: CTA groups of the batched Taylor launch (members run concurrently, one per
// group of num_sms / groups SMs); GS_ENS_GROUPS or the call's `groups` argument override it.
constexpr int kEnsembleGroups = 16;
// gs_step_ensemble_host: member chunks whose copies overlap the other chunks' steps.
constexpr int kEnsembleChunks = 4;

struct SnapSlot {
    DevBuf dev;                  // device copy of the state at the snapshot
    cudaEvent_t ready = nullptr; // the device copy is complete (recorded on the compute stream)
    bool busy = false;
};

struct SnapJob {
    int slot = 0;
    std::FILE* f = nullptr;
    std::string path;
    double origin[3] = {0, 0, 0};
    std::vector<uint8_t> labels;
};

}  // namespace

namespace gsio {
void set_free_error(const std::string& msg) { g_create_error = msg; }
}  // namespace gsio

struct gs_ctx {
    int device = 0;
    int nx = 0, ny = 0, nz = 0;
    double h = 1.0;
    int64_t n = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 0;
    int capacity = 0;  // co-resident CTAs of taylor_kernel

    // operator
    DevBuf pal, dvox, wtab, dtab;   // palette indices, fp64 D (fallback), w table, D table
    bool has_operator = false;
    bool palette_mode = true;
    bool has_labels = false;        // pal holds Material codes (0..3)
    std::vector<double> dtab_host;  // palette D values
    double anorm = 0.0;
    bool anorm_valid = false;

    // generic CSR operator (gs_create_csr)
    bool is_csr = false;
    DevBuf csr_offs, csr_cols, csr_vals, csc_offs, csc_abs;

    // vectors
    DevBuf u, g, f0, f1, t0, t1, out;
    // scratch
    DevBuf part_b, part_c, part_u, slots, mslots, xchg, x2d, ctrl, metrics, infos, normbits;
    int cap2d = 0;  // CTAs of the resident 2-D Taylor kernel the device holds at once
    // exact sequential sums (gs_seqsum.cuh): tile sums/prefixes, per-CTA item lists, counts
    DevBuf seq_tsum, seq_items, seq_counts;
    // gs_run_ensemble (this context as member 0): the members' SolveParams and the group control words
    DevBuf ens_params, ens_ctl;
    // gs_step_ensemble_host: copy streams and chunk events
    cudaStream_t ens_h2d = nullptr, ens_d2h = nullptr;
    std::vector<cudaEvent_t> ens_events;

    gs::StencilOp op{};
    int grid_blocks = 0;
    // gs_step_host: the state's H2D / D2H ride in the launch sequence (one synchronisation)
    const double* stage_in = nullptr;
    double* stage_out = nullptr;
    // value-semantics calls (gs_step_host, gs_step_ensemble_host): the step's state lives in the
    // `out` buffer (free in run mode) instead of the resident u, which stays untouched
    bool stage_swap = false;
    // one caller at a time per context (recursive: entry points call each other)
    std::recursive_mutex call_mu;
    // small-grid path (gs_cluster.cu): one 16-CTA cluster runs whole gs_run calls
    int64_t cl_slice = 0, cl_halo = 0;
    size_t cl_smem = 0;
    bool cluster_ok = false;
    bool tma_ok = false;          // TMA descriptors built (nx % 16 == 0)
    CUtensorMap xmap[gs::kNumBufs];
    CUtensorMap omap[gs::kNumBufs];
    CUtensorMap x2map[gs::kNumBufs];
    CUtensorMap x3map[gs::kNumBufs];
    CUtensorMap b3map;
    CUtensorMap lmap, l2map, l3map;
    int trace_cap = 0;
    bool ktime = false;
    double kms[4] = {0, 0, 0, 0};
    int kcount[4] = {0, 0, 0, 0};
    std::vector<cudaEvent_t> events;
    DevBuf trace;
    std::vector<uint64_t> trace_host;
    std::string err;

    // snapshot pipeline
    SnapSlot snap[kSnapSlots];
    cudaStream_t snap_stream = nullptr;  // the writer thread's stream (formatting + D2H)
    // writer-thread scratch (the writer handles one snapshot at a time)
    DevBuf fmt_lens, fmt_offs, fmt_text, fmt_tmp, fmt_tie, fmt_lab, fmt_ltext;
    char* host_text = nullptr;           // pinned: the formatted value lines, then the label lines
    double* host_u = nullptr;            // pinned: raw values for the host formatter fallback
    unsigned long long* host_small = nullptr;  // pinned: tie flag, last offset, last length
    std::thread snap_thread;
    std::mutex snap_mu;
    std::condition_variable snap_cv;
    std::deque<SnapJob> snap_q;
    bool snap_stop = false;
    gs_status snap_code = GS_OK;
    std::string snap_err;
};

namespace {

gs_status fail(gs_ctx* c, gs_status code, const std::string& msg) {
    if (c) {
        c->err = msg;
        t_err = msg;
        t_err_ctx = c;
    } else {
        g_create_error = msg;
    }
    return code;
}

// Serialise the calls on one context (the reference's operators are safe to share read-only
// across threads, SPEC.md: a context serialises instead of racing on its scratch buffers).
#define GS_LOCK(c)                                     \
    std::unique_lock<std::recursive_mutex> gs_lock_;   \
    if (c) gs_lock_ = std::unique_lock<std::recursive_mutex>((c)->call_mu)

// All members' locks, in address order (no lock-order inversion between two ensemble calls).
struct MultiLock {
    std::vector<std::unique_lock<std::recursive_mutex>> locks;
    MultiLock(gs_ctx* const* ctxs, int n) {
        std::vector<gs_ctx*> v;
        for (int i = 0; ctxs && i < n; ++i)
            if (ctxs[i]) v.push_back(ctxs[i]);
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        for (gs_ctx* c : v) locks.emplace_back(c->call_mu);
    }
};

gs_status cuda_fail(gs_ctx* c, cudaError_t e, const char* where) {
    return fail(c, GS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define GS_CUDA(ctx, call)                                  \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

// Fallback-sweep decomposition (sweep_l1): tiles of 32 x (threads/32) columns; pick the
// z-chunk so the items spread evenly over the co-resident CTAs (balance first, then the
// longest chunk for z-reuse along each column).  The TMA sweep partitions tile-planes
// itself (contiguous, balanced ranges per CTA).
void plan_items(gs_ctx* c) {
    gs::StencilOp& op = c->op;
    const int ty = gs::kSolveThreads / 32;
    op.tiles_x = (c->nx + 31) / 32;
    op.tiles_y = (c->ny + ty - 1) / ty;
    const int64_t tiles = static_cast<int64_t>(op.tiles_x) * op.tiles_y;
    const int grid = std::max(1, c->capacity);
    int best_zc = 1;
    double best_score = -1.0;
    for (int zc = 1; zc <= c->nz; ++zc) {
        const int64_t chunks = (c->nz + zc - 1) / zc;
        const int64_t items = tiles * chunks;
        const int64_t rounds = (items + grid - 1) / grid;
        const double span = static_cast<double>(rounds) * zc;  // planes per CTA on the critical path
        const double eff = static_cast<double>(tiles) * c->nz / (static_cast<double>(grid) * span);
        const double score = eff * (1.0 - 1.0 / (zc + 2.0));
        if (score > best_score + 1e-9) {
            best_score = score;
            best_zc = zc;
        }
    }
    op.zc = best_zc;
    op.chunks_z = (c->nz + best_zc - 1) / best_zc;
    op.n_items = tiles * op.chunks_z;
    c->grid_blocks = grid;
}

// TMA descriptors over the x-fastest arrays: halo boxes (TX+4)x(TY+2)x1 starting two voxels
// left of / one row below the tile (out-of-bounds elements read as 0.0), own boxes TXxTYx1, labels as u8.
gs_status build_tensor_maps(gs_ctx* c) {
    c->tma_ok = false;
    if (c->nx % 16 != 0) return GS_OK;  // u8 label rows need 16-byte pitch
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return GS_OK;  // no TMA: fallback sweep
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(c->nx), static_cast<cuuint64_t>(c->ny),
                                static_cast<cuuint64_t>(c->nz)};
    const cuuint64_t st8[2] = {static_cast<cuuint64_t>(c->nx) * 8, static_cast<cuuint64_t>(c->nx) * c->ny * 8};
    const cuuint64_t st1[2] = {static_cast<cuuint64_t>(c->nx), static_cast<cuuint64_t>(c->nx) * c->ny};
    const cuuint32_t halo[3] = {gs::kXPitch, gs::kTmaTY + 2, 1};
    const cuuint32_t own[3] = {gs::kTmaTX, gs::kTmaTY, 1};
    const cuuint32_t halo2[3] = {gs::kXPitch, gs::k2XRows, 1};
    const cuuint32_t lhalo[3] = {gs::kLPitch, gs::kTmaTY + 2, 1};
    const cuuint32_t halo3[3] = {gs::k3XPitch, gs::k3XRows, 1};
    const cuuint32_t bhalo3[3] = {gs::k3XPitch, gs::k3BRows, 1};
    const cuuint32_t lhalo3[3] = {gs::kLPitch, gs::k3LRows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    DevBuf* bufs[gs::kNumBufs] = {&c->u, &c->g, &c->f0, &c->f1, &c->t0, &c->t1, &c->out};
    for (int b = 0; b < gs::kNumBufs; ++b) {
        CUresult r = encode(&c->xmap[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, bufs[b]->p, dims, st8, halo, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(halo) failed: " + std::to_string(r));
        r = encode(&c->omap[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, bufs[b]->p, dims, st8, own, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(own) failed: " + std::to_string(r));
        r = encode(&c->x2map[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, bufs[b]->p, dims, st8, halo2, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(halo2) failed: " + std::to_string(r));
        r = encode(&c->x3map[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, bufs[b]->p, dims, st8, halo3, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(halo3) failed: " + std::to_string(r));
    }
    CUresult rb = encode(&c->b3map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->g.p, dims, st8, bhalo3, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rb != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(b halo3) failed: " + std::to_string(rb));
    rb = encode(&c->l3map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, c->pal.p, dims, st1, lhalo3, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rb != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(labels halo3) failed: " + std::to_string(rb));
    CUresult r = encode(&c->lmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, c->pal.p, dims, st1, own, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(labels) failed: " + std::to_string(r));
    r = encode(&c->l2map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, c->pal.p, dims, st1, lhalo, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, GS_ECUDA, "cuTensorMapEncodeTiled(labels halo) failed: " + std::to_string(r));
    c->tma_ok = true;
    return GS_OK;
}

gs_status ensure_operator(gs_ctx* c) {
    if (!c->has_operator)
        return fail(c, GS_EINVAL, "operator not set: call gs_set_labels, gs_set_intensity or gs_set_diffusion");
    return GS_OK;
}

void fill_op(gs_ctx* c) {
    gs::StencilOp& op = c->op;
    op.nx = c->nx;
    op.ny = c->ny;
    op.nz = c->nz;
    op.n = c->n;
    op.sy = c->nx;
    op.sz = static_cast<int64_t>(c->nx) * c->ny;
    op.inv_h2 = 1.0 / (c->h * c->h);  // stencil.cpp:8
    op.pal = c->palette_mode ? c->pal.as<uint8_t>() : nullptr;
    op.dvox = c->palette_mode ? nullptr : c->dvox.as<double>();
    op.wtab = c->wtab.as<double>();
    op.csr_offs = c->is_csr ? c->csr_offs.as<int64_t>() : nullptr;
    op.csr_cols = c->is_csr ? c->csr_cols.as<int32_t>() : nullptr;
    op.csr_vals = c->is_csr ? c->csr_vals.as<double>() : nullptr;
}

// w table from palette D values: w = D * (1/(h*h)) exactly as stencil.cpp:8,23.
gs_status upload_palette(gs_ctx* c, const std::vector<double>& dvals) {
    std::vector<double> w(256, 0.0), d(256, 0.0);
    const double inv_h2 = 1.0 / (c->h * c->h);
    for (size_t k = 0; k < dvals.size(); ++k) {
        d[k] = dvals[k];
        w[k] = dvals[k] != 0.0 ? dvals[k] * inv_h2 : 0.0;
        if (dvals[k] != 0.0 && w[k] == 0.0)
            return fail(c, GS_EINVAL, "diffusion coefficient underflows D/h^2");
    }
    c->dtab_host = d;
    GS_CUDA(c, c->wtab.alloc(256 * sizeof(double)));
    GS_CUDA(c, c->dtab.alloc(256 * sizeof(double)));
    GS_CUDA(c, cudaMemcpyAsync(c->wtab.p, w.data(), 256 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    GS_CUDA(c, cudaMemcpyAsync(c->dtab.p, d.data(), 256 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    return GS_OK;
}

gs_status compute_anorm(gs_ctx* c) {
    GS_CUDA(c, c->normbits.alloc(sizeof(unsigned long long)));
    GS_CUDA(c, cudaMemsetAsync(c->normbits.p, 0, sizeof(unsigned long long), c->stream));
    const int blocks = static_cast<int>(std::min<int64_t>((c->n + 255) / 256, 148 * 8));
    if (c->is_csr)
        gs::csc_norm_kernel<<<std::max(1, blocks), 256, 0, c->stream>>>(c->n, c->csc_offs.as<int64_t>(),
                                                                         c->csc_abs.as<double>(),
                                                                         c->normbits.as<unsigned long long>());
    else
        gs::colsum_norm_kernel<<<std::max(1, blocks), 256, 0, c->stream>>>(c->op, c->normbits.as<unsigned long long>());
    GS_CUDA(c, cudaGetLastError());
    unsigned long long bits = 0;
    GS_CUDA(c, cudaMemcpyAsync(&bits, c->normbits.p, sizeof bits, cudaMemcpyDeviceToHost, c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    double v;
    std::memcpy(&v, &bits, sizeof v);
    c->anorm = v;
    c->anorm_valid = true;
    return GS_OK;
}

// The cluster kernel's dynamic shared-memory limit is a per-function attribute shared by every
// context in the process: it only ever grows (to the largest grid's need), so a context created
// later for a smaller grid cannot invalidate the launches of an earlier, larger one.
bool raise_cluster_smem(size_t smem) {
    static std::mutex mu;
    static size_t cur = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (smem <= cur) return true;
    if (cudaFuncSetAttribute(gs::cluster_run_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
        return false;
    cur = smem;
    return true;
}

gs_status operator_ready(gs_ctx* c) {
    c->has_operator = true;
    c->anorm_valid = false;
    fill_op(c);
    return compute_anorm(c);
}

// r_m for m = 1..55 with glibc, exactly expact.cpp:47-48.
void fill_rtab(double tol, double* rtab) {
    rtab[0] = 0.0;
    for (int m = 1; m <= gs::kMaxDegree; ++m) {
        double r = std::exp((std::log(tol) + std::lgamma(m + 2.0)) / (m + 1.0));
        rtab[m] = (6.0 < r) ? 6.0 : r;  // std::min(r, r_cap)
    }
}

// Grid sizes of the launch sequence.  prep/taylor: one CTA per SM (the TMA rings take most
// of shared memory); border/update/metrics: streaming kernels, two CTAs per SM.
// Small grids get fewer streaming CTAs (>= 8 voxels per thread): their per-block reductions,
// tickets and partial-sum trees cost more than the sweep itself at 32^3.
int stream_blocks(const gs_ctx* c) {
    const int64_t want = (c->n + 8 * gs::kSolveThreads - 1) / (8 * gs::kSolveThreads);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 2 * c->num_sms)));
}

// Lockstep work split of the TMA sweeps (gs::cta_work): with P tiles per plane and a grid
// of G >= P CTAs, k = G / P groups of P CTAs march z-chunks of [0, zm) one tile each, and
// the E = G - kP others split the slab [zm, nz).  zm balances the two: a group CTA streams
// zm/k planes, an extra CTA P(nz - zm)/E planes in about P/E + 1 segments, each segment
// costing c0 planes more (its z-halo planes and prologue).  GS_LOCK=0 restores the even
// split; GS_LOCK_C0 overrides c0.
void lockstep_split(const gs_ctx* c, int gb, gs::SolveParams& p) {
    p.lock_groups = 0;
    p.lock_zm = 0;
    if (!p.use_tma || p.fuse == 4) return;
    if (const char* e = std::getenv("GS_LOCK"))
        if (std::atoi(e) == 0) return;
    const int64_t P = static_cast<int64_t>((c->nx + gs::kTmaTX - 1) / gs::kTmaTX) * ((c->ny + gs::kTmaTY - 1) / gs::kTmaTY);
    const int64_t k = gb / P;
    if (k < 1 || c->nz < 8 * k) return;
    const int64_t E = gb - k * P;
    // c0 measured with 32 x 32 tiles (steps/s, c0 = 3 / 6 / 9 / 12): C4 (nz 256) 96.3 / 97.5 /
    // 96.7 / 96.1, C3 (nz 128) 1660 / 1645 / 1643 / 1646
    double c0 = c->nz >= 192 ? 6.0 : 3.0;
    if (const char* e = std::getenv("GS_LOCK_C0")) c0 = std::atof(e);
    int64_t zm = c->nz;
    if (E > 0) {
        const double z = (static_cast<double>(P) * c->nz + c0 * P) / (static_cast<double>(E) / k + P);
        zm = std::min<int64_t>(c->nz, std::max<int64_t>(k, std::llround(z)));
        if (P * (c->nz - zm) < E) zm = c->nz;
    }
    p.lock_groups = static_cast<int>(k);
    p.lock_zm = static_cast<int>(zm);
}

int tiles_2d(const gs_ctx* c) { return ((c->nx + 31) / 32) * ((c->ny + 31) / 32); }

// The cooperative Taylor launch of one step: the resident-tile kernel on 2-D grids, else the
// TMA sweeps on gb CTAs.
cudaError_t launch_taylor(gs_ctx* c, const gs::SolveParams& p, int gb, void** args) {
    if (p.use_2d)
        return cudaLaunchCooperativeKernel(gs::taylor2d_kernel_fn(), dim3(p.use_2d), dim3(gs::kSolveThreads), args,
                                           gs::k2dSmemBytes, c->stream);
    return cudaLaunchCooperativeKernel(gs::taylor_kernel_fn(p.fuse), dim3(gb), dim3(gs::kSolveThreads), args,
                                       gs::kDynSmemBytes, c->stream);
}

// Scratch, state staging and the context-dependent SolveParams fields of one run on the
// context's stream: gb CTAs for prep / taylor, sb for the streaming kernels.
gs_status setup_solve(gs_ctx* c, gs::SolveParams& p, int gb, int sb, int n_steps, gs_metrics* metrics,
                      gs_step_info* infos) {
    const int pb = std::max(gb, sb);
    GS_CUDA(c, c->part_b.alloc(sizeof(double) * pb));
    GS_CUDA(c, c->part_c.alloc(sizeof(double) * pb));
    GS_CUDA(c, c->part_u.alloc(sizeof(double) * pb));
    GS_CUDA(c, c->slots.alloc(sizeof(unsigned long long) * gs::kSlotWords));
    GS_CUDA(c, c->mslots.alloc(sizeof(unsigned long long) * 4));
    const bool fresh_ctrl = c->ctrl.p == nullptr;
    GS_CUDA(c, c->ctrl.alloc(sizeof(gs::Ctrl)));
    GS_CUDA(c, cudaMemsetAsync(c->slots.p, 0, sizeof(unsigned long long) * gs::kSlotWords, c->stream));
    GS_CUDA(c, c->xchg.alloc(sizeof(unsigned long long) * gs::kXchgWords));
    GS_CUDA(c, cudaMemsetAsync(c->xchg.p, 0, sizeof(unsigned long long) * gs::kXchgWords, c->stream));
    const unsigned long long ms_init[4] = {0ull, ~0ull, 0ull, 0ull};
    GS_CUDA(c, cudaMemcpyAsync(c->mslots.p, ms_init, sizeof ms_init, cudaMemcpyHostToDevice, c->stream));
    // a new run starts from a clean control block, except last_terms (the previous call's
    // Taylor terms, which orders the next ensemble queue): it is the last field
    GS_CUDA(c, cudaMemsetAsync(c->ctrl.p, 0, fresh_ctrl ? sizeof(gs::Ctrl) : offsetof(gs::Ctrl, last_terms),
                               c->stream));
    if (c->stage_in)
        GS_CUDA(c, cudaMemcpyAsync(c->stage_swap ? c->out.p : c->u.p, c->stage_in, sizeof(double) * static_cast<size_t>(c->n),
                                   cudaMemcpyHostToDevice, c->stream));
    if (metrics) GS_CUDA(c, c->metrics.alloc(sizeof(double) * 4 * (n_steps + 1)));
    if (infos) {
        GS_CUDA(c, c->infos.alloc(sizeof(gs_step_info) * std::max(1, n_steps)));
        GS_CUDA(c, cudaMemsetAsync(c->infos.p, 0, sizeof(gs_step_info) * std::max(1, n_steps), c->stream));
    }
    p.op = c->op;
    p.grid_blocks = gb;
    p.anorm = c->anorm;
    p.use_tma = (c->tma_ok && c->palette_mode && !c->is_csr && std::getenv("GS_DISABLE_TMA") == nullptr) ? 1 : 0;
    if (p.use_tma) {
        for (int b = 0; b < gs::kNumBufs; ++b) {
            p.xmap[b] = c->xmap[b];
            p.omap[b] = c->omap[b];
            p.x2map[b] = c->x2map[b];
            p.x3map[b] = c->x3map[b];
        }
        p.b3map = c->b3map;
        p.lmap = c->lmap;
        p.l2map = c->l2map;
        p.l3map = c->l3map;
    }
    // Taylor terms per fused sweep (GS_FUSE=2|3 overrides the default for A/B measurements)
    p.fuse = kDefaultFuse;
    if (const char* f = std::getenv("GS_FUSE")) p.fuse = std::atoi(f) == 3 ? 3 : 2;
    // thin grids (2-D and a few planes): the two-term sweep that skips the planes past the grid
    if (p.fuse == 2 && c->nz < 8) p.fuse = 4;
    lockstep_split(c, gb, p);
    // GS_EXACT_MAX=1|2: test modes of the two-term sweeps' maxima (see taylor_kernel)
    p.exact_max = 0;
    if (const char* e = std::getenv("GS_EXACT_MAX")) p.exact_max = std::atoi(e);
    p.metrics =metrics ? c->metrics.as<double>() : nullptr;
    p.want_metrics = metrics ? 1 : 0;
    p.infos = infos ? c->infos.as<gs_step_info>() : nullptr;
    p.part_b = c->part_b.as<double>();
    p.part_c = c->part_c.as<double>();
    p.part_u = c->part_u.as<double>();
    p.slots = c->slots.as<unsigned long long>();
    p.mslots = c->mslots.as<unsigned long long>();
    // GS_NO_XCHG=1: the atomicMax slots and the plain grid barrier (A/B)
    p.xchg = (gb <= gs::kXchgCtas && std::getenv("GS_NO_XCHG") == nullptr) ? c->xchg.as<unsigned long long>() : nullptr;
    // 2-D grids whose 32 x 32 tiles all fit the device at once: the resident-tile Taylor kernel
    // (gs_flat2d.cuh); GS_NO_2D=1 keeps them on the TMA sweeps (A/B, tests)
    p.use_2d = 0;
    p.x2d = nullptr;
    {
        const int t2d = tiles_2d(c);
        if (gs_uses_flat2d(c)) {
            GS_CUDA(c, c->x2d.alloc(sizeof(double) * 2 * (gs::k2dK + 1) * static_cast<size_t>(c->n)));
            p.use_2d = t2d;
            p.x2d = c->x2d.as<double>();
        }
    }
    p.ctrl = c->ctrl.as<gs::Ctrl>();
    // the reference's sequential ||b||_1 and bordered column sum (GS_TREE_SUMS=1: tree sums, A/B)
    p.seq_exact = std::getenv("GS_TREE_SUMS") == nullptr ? (std::getenv("GS_SEQ_DEBUG") ? 2 : 1) : 0;
    p.seq_tiles = static_cast<int>((c->n + gs::kSeqTileElems - 1) / gs::kSeqTileElems);
    GS_CUDA(c, c->seq_tsum.alloc(sizeof(double) * 2 * std::max(1, p.seq_tiles)));  // tile sums, then prefixes
    {
        const int sq = std::min(2 * c->num_sms, gs::kSeqMaxCtas);  // >= any seq_ctas()
        GS_CUDA(c, c->seq_items.alloc(static_cast<size_t>(gs::kSeqItemBytes) * gs::kSeqItemsPerCta * sq));
        GS_CUDA(c, c->seq_counts.alloc(sizeof(int) * 2 * sq));
    }
    p.seq_tsum = c->seq_tsum.as<double>();
    p.seq_items = c->seq_items.p;
    p.seq_counts = c->seq_counts.as<int>();
    DevBuf* bufs[gs::kNumBufs] = {&c->u, &c->g, &c->f0, &c->f1, &c->t0, &c->t1, &c->out};
    for (int b = 0; b < gs::kNumBufs; ++b) p.buf[b] = bufs[b]->as<double>();
    if (c->stage_swap) {  // the state is the staging (`out`) buffer: pointer and TMA maps
        p.buf[gs::kBufU] = c->out.as<double>();
        if (p.use_tma) {
            p.xmap[gs::kBufU] = c->xmap[gs::kBufOut];
            p.omap[gs::kBufU] = c->omap[gs::kBufOut];
            p.x2map[gs::kBufU] = c->x2map[gs::kBufOut];
            p.x3map[gs::kBufU] = c->x3map[gs::kBufOut];
        }
    }
    p.trace = nullptr;
    p.trace_cap = 0;
    if (c->trace_cap > 0) {
        GS_CUDA(c, c->trace.alloc(sizeof(uint64_t) * 2 * c->trace_cap));
        GS_CUDA(c, cudaMemsetAsync(c->trace.p, 0, sizeof(uint64_t) * 2 * c->trace_cap, c->stream));
        p.trace = c->trace.as<unsigned long long>();
        p.trace_cap = c->trace_cap;
    }
    return GS_OK;
}

// CTAs of the prep / Taylor launches: one per SM, capped at the TMA sweeps' tile-plane count
// (CTAs beyond it would only join the grid barriers; C1/C2: 64 tile-planes, 64 CTAs run
// 8-10% faster than 148).
int solve_blocks(const gs_ctx* c) {
    int gb = c->grid_blocks;
    if (const char* e = std::getenv("GS_GRID"))  // A/B of the CTA count (capped at co-residency)
        gb = std::max(1, std::min(gb, std::atoi(e)));
    if (c->tma_ok && c->palette_mode && !c->is_csr) {
        const int64_t q = static_cast<int64_t>((c->nx + gs::kTmaTX - 1) / gs::kTmaTX) *
                          ((c->ny + gs::kTmaTY - 1) / gs::kTmaTY) * c->nz;
        gb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(gb, q)));
    }
    return gb;
}

// The exact sequential sum `which` (0: ||b||_1 before the border pass, 1: the bordered column
// sum after it) on the context's stream; expmv has neither.
// CTAs of the seqsum kernels for one run when `members` runs share the GPU: about two per SM
// in all (one resident wave), at least a few tiles each; GS_SEQ_CTAS overrides (A/B).
int seq_ctas(const gs_ctx* c, int tiles, int members) {
    int k = 2 * c->num_sms;
    (void)members;
    if (const char* e = std::getenv("GS_SEQ_CTAS")) k = std::max(1, std::atoi(e));
    return std::max(1, std::min({k, (tiles + 1) / 2, 2 * c->num_sms, gs::kSeqMaxCtas}));
}

void launch_seqsum(gs_ctx* c, const gs::SolveParams& p, int which) {
    if (!p.seq_exact || p.mode == gs::kModeExpmv) return;
    const int k = seq_ctas(c, p.seq_tiles, 1);
    // the tile pass: one CTA per SM at most (its last-CTA ticket costs ~50 ns per CTA; measured
    // C3 14.5 us with 148 CTAs against 21 us with 256 and 35 us with 592)
    int k1 = std::max(1, std::min(p.seq_tiles, c->num_sms));
    if (const char* e = std::getenv("GS_SEQ_CTAS1")) k1 = std::max(1, std::min(p.seq_tiles, std::atoi(e)));
    gs::seqsum_tiles_kernel<<<k1, gs::kSolveThreads, 0, c->stream>>>(p, which);
    gs::seqsum_items_kernel<<<k, gs::kSolveThreads, 0, c->stream>>>(p, which);
}

gs_status launch_solve(gs_ctx* c, gs::SolveParams& p, int n_steps, gs_metrics* metrics, gs_step_info* infos) {
    const int gb = solve_blocks(c);       // prep / taylor (co-resident)
    const int sb = stream_blocks(c);      // border / update / metrics
    {
        const gs_status st = setup_solve(c, p, gb, sb, n_steps, metrics, infos);
        if (st != GS_OK) return st;
    }
    const size_t dyn = gs::kDynSmemBytes;  // the Taylor kernel's reduction scratch is dynamic (kRedOffset)
    const size_t dyn_prep = p.use_tma ? gs::kRingBytes : 0;
    const dim3 blk(gs::kSolveThreads);
    // optional per-kernel CUDA-event timing: record (kind, start, end) around each launch
    std::vector<std::pair<int, int>> marks;  // (kind, event index of start)
    auto ev = [&](int k) -> cudaError_t {
        if (!c->ktime) return cudaSuccess;
        const size_t need = 2 * (marks.size() + 1);
        while (c->events.size() < need) {
            cudaEvent_t e;
            cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return r;
            c->events.push_back(e);
        }
        marks.push_back({k, static_cast<int>(2 * marks.size())});
        return cudaEventRecord(c->events[marks.back().second], c->stream);
    };
    auto ev_end = [&]() -> cudaError_t {
        if (!c->ktime) return cudaSuccess;
        return cudaEventRecord(c->events[marks.back().second + 1], c->stream);
    };
    const bool use_cluster = p.mode == gs::kModeRun && c->cluster_ok && c->palette_mode && !c->is_csr &&
                             std::getenv("GS_NO_CLUSTER") == nullptr;
    if (use_cluster) {
        gs::ClusterParams cp{};
        cp.op = c->op;
        cp.n_steps = n_steps;
        cp.want_metrics = metrics ? 1 : 0;
        cp.seq_exact = p.seq_exact;
        cp.slice = c->cl_slice;
        cp.halo = c->cl_halo;
        cp.rho = p.rho;
        cp.tau = p.tau;
        cp.tol = p.tol;
        cp.anorm = c->anorm;
        std::copy(p.rtab, p.rtab + gs::kMaxDegree + 1, cp.rtab);
        cp.u = p.buf[gs::kBufU];
        cp.metrics = p.metrics;
        cp.infos = p.infos;
        cp.ctrl = p.ctrl;
        for (int a = 0; a < 3; ++a) {
            cp.origin[a] = p.origin[a];
            cp.center[a] = p.center[a];
        }
        cp.h = p.h;
        cp.front_threshold = p.front_threshold;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(gs::kClusterCTAs);
        cfg.blockDim = dim3(gs::kSolveThreads);
        cfg.dynamicSmemBytes = c->cl_smem;
        cfg.stream = c->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = gs::kClusterCTAs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        GS_CUDA(c, ev(2));  // timed as the Taylor kernel: it is the whole step here
        GS_CUDA(c, cudaLaunchKernelEx(&cfg, gs::cluster_run_kernel, cp));
        GS_CUDA(c, ev_end());
    } else if (p.mode == gs::kModeApply) {
        GS_CUDA(c, ev(0));
        gs::prep_kernel<<<gb, blk, dyn_prep, c->stream>>>(p, 0);
        GS_CUDA(c, cudaGetLastError());
        GS_CUDA(c, ev_end());
    } else {
        const int steps = p.mode == gs::kModeRun ? n_steps : 1;
        if (p.mode == gs::kModeRun && metrics) {
            gs::metrics_kernel<<<sb, blk, 0, c->stream>>>(p);
            GS_CUDA(c, cudaGetLastError());
        }
        // Runs of several steps replay one captured step as a CUDA graph: the four kernels'
        // ~4 KB parameter blocks are uploaded once, and the step index lives on the device
        // (advance_kernel).  Timing/trace modes and a failed capture use direct launches.
        bool graphed = false;
        if (p.mode == gs::kModeRun && steps >= 2 && !c->ktime && c->trace_cap == 0 &&
            std::getenv("GS_NO_GRAPH") == nullptr) {
            cudaGraph_t graph = nullptr;
            cudaGraphExec_t exec = nullptr;
            int border_blocks = sb, neg = -1;
            void* args[] = {&p, &border_blocks, &neg};
            bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                gs::prep_kernel<<<gb, blk, dyn_prep, c->stream>>>(p, -1);
                launch_seqsum(c, p, 0);
                gs::border_kernel<<<sb, blk, 0, c->stream>>>(p, gb, -1);
                launch_seqsum(c, p, 1);
                launch_taylor(c, p, gb, args);
                gs::update_kernel<<<sb, blk, 0, c->stream>>>(p, -1);
                gs::advance_kernel<<<1, 1, 0, c->stream>>>(p.ctrl);
                ok = cudaStreamEndCapture(c->stream, &graph) == cudaSuccess && graph != nullptr;
                ok = ok && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
            }
            cudaError_t le = cudaSuccess;
            if (ok) {
                for (int step = 0; step < steps && le == cudaSuccess; ++step) le = cudaGraphLaunch(exec, c->stream);
                graphed = true;
            } else {
                cudaGetLastError();  // nothing ran during the capture: fall back to direct launches
            }
            if (graphed && le == cudaSuccess) le = cudaStreamSynchronize(c->stream);  // before destroying
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
            GS_CUDA(c, le);
        }
        for (int step = 0; step < steps && !graphed; ++step) {
            GS_CUDA(c, ev(0));
            gs::prep_kernel<<<gb, blk, dyn_prep, c->stream>>>(p, step);
            GS_CUDA(c, cudaGetLastError());
            GS_CUDA(c, ev_end());
            GS_CUDA(c, ev(1));  // border and the two exact sums
            launch_seqsum(c, p, 0);
            gs::border_kernel<<<sb, blk, 0, c->stream>>>(p, gb, step);
            launch_seqsum(c, p, 1);
            GS_CUDA(c, cudaGetLastError());
            GS_CUDA(c, ev_end());
            int border_blocks = sb;
            void* args[] = {&p, &border_blocks, &step};
            GS_CUDA(c, ev(2));
            GS_CUDA(c, launch_taylor(c, p, gb, args));
            GS_CUDA(c, ev_end());
            GS_CUDA(c, ev(3));
            gs::update_kernel<<<sb, blk, 0, c->stream>>>(p, step);
            GS_CUDA(c, cudaGetLastError());
            GS_CUDA(c, ev_end());
        }
    }
    if (c->stage_out)
        GS_CUDA(c, cudaMemcpyAsync(c->stage_out, p.buf[gs::kBufU], sizeof(double) * static_cast<size_t>(c->n),
                                   cudaMemcpyDeviceToHost, c->stream));
    gs::Ctrl ctrl{};
    GS_CUDA(c, cudaMemcpyAsync(&ctrl, c->ctrl.p, sizeof ctrl, cudaMemcpyDeviceToHost, c->stream));
    if (metrics)
        GS_CUDA(c, cudaMemcpyAsync(metrics, c->metrics.p, sizeof(double) * 4 * (n_steps + 1), cudaMemcpyDeviceToHost,
                                   c->stream));
    if (infos)
        GS_CUDA(c, cudaMemcpyAsync(infos, c->infos.p, sizeof(gs_step_info) * std::max(1, n_steps),
                                   cudaMemcpyDeviceToHost, c->stream));
    if (c->trace_cap > 0) {
        c->trace_host.assign(2 * static_cast<size_t>(c->trace_cap), 0);
        GS_CUDA(c, cudaMemcpyAsync(c->trace_host.data(), c->trace.p, sizeof(uint64_t) * 2 * c->trace_cap,
                                   cudaMemcpyDeviceToHost, c->stream));
    }
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->ktime) {
        for (int k = 0; k < 4; ++k) {
            c->kms[k] = 0.0;
            c->kcount[k] = 0;
        }
        for (const auto& m : marks) {
            float ms = 0.f;
            GS_CUDA(c, cudaEventElapsedTime(&ms, c->events[m.second], c->events[m.second + 1]));
            c->kms[m.first] += ms;
            c->kcount[m.first] += 1;
        }
    }
    if (ctrl.status != GS_OK) {
        if (ctrl.detail == 2) return fail(c, GS_ENUMERIC, "expmv: series diverged to non-finite values; reduce t");
        if (ctrl.status == GS_EINVAL)
            return fail(c, GS_EINVAL, "select_params: operator norm must be finite and nonnegative");
        return fail(c, GS_ENUMERIC, "select_params: scaled operator norm too large for any stage count");
    }
    return GS_OK;
}

bool tol_ok(double tol) { return tol > 0.0 && tol < 1.0; }

}  // namespace

namespace {

// One snapshot job on the writer thread: the value column formatted on the GPU (gs_vtkfmt.cu),
// the material column too when every code is < 10, the text copied back and written.  A value
// the GPU formatter flags (near a rounding tie), or a grid too large for it, goes through the
// host formatter instead; either way the bytes are write_vtk's (vtk.cpp:59-91).
bool snapshot_write_job(gs_ctx* c, SnapJob& j, gsio::Error& err) {
    SnapSlot& s = c->snap[j.slot];
    const int64_t n = c->n;
    const bool with_labels = !j.labels.empty();
    auto cuda_err = [&](cudaError_t e) {
        err = {GS_ECUDA, std::string("gs_snapshot_vtk: ") + cudaGetErrorString(e)};
        return false;
    };
    cudaError_t e = cudaSuccess;
    if (!c->snap_stream) e = cudaStreamCreateWithFlags(&c->snap_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && !c->host_small) e = cudaMallocHost(&c->host_small, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->snap_stream, s.ready, 0);
    if (e != cudaSuccess) return cuda_err(e);
    bool labels_on_gpu = with_labels;
    for (size_t v = 0; labels_on_gpu && v < j.labels.size(); ++v) labels_on_gpu = j.labels[v] < 10;
    bool gpu = n < (int64_t{1} << 31) && std::getenv("GS_HOST_VTK") == nullptr;
    if (gpu) {
        gs::VtkfmtScratch sc;
        const size_t scan = gs::vtkfmt_scratch_bytes(n);
        e = gs::vtkfmt_init();
        if (e == cudaSuccess) e = c->fmt_lens.alloc(8 * static_cast<size_t>(n));
        if (e == cudaSuccess) e = c->fmt_offs.alloc(8 * static_cast<size_t>(n));
        if (e == cudaSuccess) e = c->fmt_text.alloc(static_cast<size_t>(gs::kVtkMaxLine) * n);
        if (e == cudaSuccess) e = c->fmt_tmp.alloc(std::max<size_t>(scan, 16));
        if (e == cudaSuccess) e = c->fmt_tie.alloc(sizeof(int));
        if (e == cudaSuccess && labels_on_gpu) e = c->fmt_lab.alloc(static_cast<size_t>(n));
        if (e == cudaSuccess && labels_on_gpu) e = c->fmt_ltext.alloc(2 * static_cast<size_t>(n));
        if (e == cudaSuccess && !c->host_text)
            e = cudaMallocHost(&c->host_text, static_cast<size_t>(gs::kVtkMaxLine + 2) * n);
        if (e != cudaSuccess) return cuda_err(e);
        sc.lens = c->fmt_lens.as<unsigned long long>();
        sc.offs = c->fmt_offs.as<unsigned long long>();
        sc.text = c->fmt_text.as<char>();
        sc.scan_tmp = c->fmt_tmp.p;
        sc.scan_bytes = std::max<size_t>(scan, 16);
        sc.tie = c->fmt_tie.as<int>();
        e = gs::vtkfmt_values(s.dev.as<double>(), n, sc, c->snap_stream);
        if (e == cudaSuccess && labels_on_gpu) {
            e = cudaMemcpyAsync(c->fmt_lab.p, j.labels.data(), static_cast<size_t>(n), cudaMemcpyHostToDevice,
                                c->snap_stream);
            if (e == cudaSuccess) e = gs::vtkfmt_labels(c->fmt_lab.as<uint8_t>(), n, c->fmt_ltext.as<char>(), c->snap_stream);
        }
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(c->host_small, sc.tie, sizeof(int), cudaMemcpyDeviceToHost, c->snap_stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(c->host_small + 1, sc.offs + (n - 1), 8, cudaMemcpyDeviceToHost, c->snap_stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(c->host_small + 2, sc.lens + (n - 1), 8, cudaMemcpyDeviceToHost, c->snap_stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->snap_stream);
        if (e != cudaSuccess) return cuda_err(e);
        gpu = *reinterpret_cast<const int*>(c->host_small) == 0;  // no near-tie value
        if (gpu) {
            const size_t total = static_cast<size_t>(c->host_small[1] + c->host_small[2]);
            e = cudaMemcpyAsync(c->host_text, sc.text, total, cudaMemcpyDeviceToHost, c->snap_stream);
            if (e == cudaSuccess && labels_on_gpu)
                e = cudaMemcpyAsync(c->host_text + total, c->fmt_ltext.p, 2 * static_cast<size_t>(n),
                                    cudaMemcpyDeviceToHost, c->snap_stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(c->snap_stream);
            if (e != cudaSuccess) return cuda_err(e);
            const std::string head = gsio::vtk_header(c->nx, c->ny, c->nz, c->h, j.origin);
            bool ok = std::fwrite(head.data(), 1, head.size(), j.f) == head.size();
            ok = ok && std::fwrite(c->host_text, 1, total, j.f) == total;
            if (ok && with_labels) {
                const size_t lh = std::strlen(gsio::kVtkMaterialHead);
                ok = std::fwrite(gsio::kVtkMaterialHead, 1, lh, j.f) == lh;
                if (ok && labels_on_gpu) {
                    ok = std::fwrite(c->host_text + total, 1, 2 * static_cast<size_t>(n), j.f) ==
                         2 * static_cast<size_t>(n);
                } else if (ok) {  // codes >= 10: the host formats the material column
                    std::string t;
                    for (uint8_t code : j.labels) t += std::to_string(code) + '\n';
                    ok = std::fwrite(t.data(), 1, t.size(), j.f) == t.size();
                }
            }
            ok = ok && std::fflush(j.f) == 0;
            if (!ok) err = {GS_EDATA, "write failed: " + j.path};
            return ok;
        }
    }
    // host formatter: raw values back, then the parallel exact %.17g writer
    if (!c->host_u) e = cudaMallocHost(&c->host_u, sizeof(double) * static_cast<size_t>(n));
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->host_u, s.dev.p, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                            c->snap_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->snap_stream);
    if (e != cudaSuccess) return cuda_err(e);
    return gsio::write_vtk_stream(j.f, j.path, c->host_u, c->nx, c->ny, c->nz, c->h, j.origin,
                                  with_labels ? j.labels.data() : nullptr, 0, err);
}

void snapshot_writer(gs_ctx* c) {
    cudaSetDevice(c->device);
    for (;;) {
        SnapJob j;
        {
            std::unique_lock<std::mutex> lk(c->snap_mu);
            c->snap_cv.wait(lk, [&] { return c->snap_stop || !c->snap_q.empty(); });
            if (c->snap_q.empty()) return;  // stop requested and nothing left
            j = std::move(c->snap_q.front());
            c->snap_q.pop_front();
        }
        gsio::Error err;
        bool ok = snapshot_write_job(c, j, err);
        if (std::fclose(j.f) != 0 && ok) {
            ok = false;
            err = {GS_EDATA, "write failed: " + j.path};
        }
        {
            std::lock_guard<std::mutex> lk(c->snap_mu);
            c->snap[j.slot].busy = false;
            if (!ok && c->snap_code == GS_OK) {
                c->snap_code = static_cast<gs_status>(err.code);
                c->snap_err = err.msg;
            }
        }
        c->snap_cv.notify_all();
    }
}

}  // namespace

extern "C" {

gs_status gs_create(gs_ctx** out, int nx, int ny, int nz, double h, int device) {
    if (!out) return fail(nullptr, GS_EINVAL, "gs_create: null output pointer");
    *out = nullptr;
    if (nx < 1 || ny < 1 || nz < 1) return fail(nullptr, GS_EINVAL, "Grid: point counts must be >= 1");
    if (!(h > 0.0)) return fail(nullptr, GS_EINVAL, "Grid: spacing h must be positive");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, GS_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(nullptr, GS_EINVAL, "gs_create: bad device ordinal");
    gs_ctx* c = new gs_ctx();
    c->device = device;
    c->nx = nx;
    c->ny = ny;
    c->nz = nz;
    c->h = h;
    c->n = static_cast<int64_t>(nx) * ny * nz;
    auto bail = [&](cudaError_t err, const char* where) {
        g_create_error = std::string(where) + ": " + cudaGetErrorString(err);
        gs_destroy(c);
        return GS_ECUDA;
    };
    if ((e = cudaSetDevice(device)) != cudaSuccess) return bail(e, "cudaSetDevice");
    cudaDeviceProp prop{};
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return bail(e, "cudaGetDeviceProperties");
    if (prop.major != 10) {
        g_create_error = "gs_create: this build targets sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                         std::to_string(prop.minor);
        gs_destroy(c);
        return GS_ECUDA;
    }
    if (!prop.cooperativeLaunch) {
        g_create_error = "gs_create: device lacks cooperative launch";
        gs_destroy(c);
        return GS_ECUDA;
    }
    c->num_sms = prop.multiProcessorCount;
    for (const void* fn : {gs::taylor_kernel_fn(2), gs::taylor_kernel_fn(3), gs::taylor_kernel_fn(4)})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, gs::kDynSmemBytes)) != cudaSuccess)
            return bail(e, "cudaFuncSetAttribute(smem)");
    for (const void* fn : {gs::ens_taylor_kernel_fn(2), gs::ens_taylor_kernel_fn(4)})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, gs::kDynSmemBytes)) != cudaSuccess)
            return bail(e, "cudaFuncSetAttribute(smem ens)");
    // prep sweeps with the single-term ring only
    for (const void* fn : {reinterpret_cast<const void*>(gs::prep_kernel), reinterpret_cast<const void*>(gs::ens_prep_kernel)})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, gs::kRingBytes)) != cudaSuccess)
            return bail(e, "cudaFuncSetAttribute(smem prep)");
    if (const void* fn2 = gs::taylor2d_kernel_fn()) {
        if ((e = cudaFuncSetAttribute(fn2, cudaFuncAttributeMaxDynamicSharedMemorySize, gs::k2dSmemBytes)) != cudaSuccess)
            return bail(e, "cudaFuncSetAttribute(smem 2d)");
        int per2 = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, fn2, gs::kSolveThreads, gs::k2dSmemBytes)) !=
            cudaSuccess)
            return bail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor(2d)");
        c->cap2d = per2 * c->num_sms;
    }
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs::taylor_kernel_fn(2), gs::kSolveThreads,
                                                           gs::kDynSmemBytes)) != cudaSuccess)
        return bail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    int per_sm3 = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, gs::taylor_kernel_fn(3), gs::kSolveThreads,
                                                           gs::kDynSmemBytes)) != cudaSuccess)
        return bail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    per_sm = std::min(per_sm, per_sm3);
    if (per_sm < 1) {
        g_create_error = "gs_create: solve kernel does not fit on an SM";
        gs_destroy(c);
        return GS_ECUDA;
    }
    c->capacity = per_sm * c->num_sms;
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "cudaStreamCreate");
    {
        // The whole state fits one cluster when every CTA's slice holds at least one halo
        // (one plane, or one row in 2-D) and the slices fit in shared memory.
        const int64_t sy = nx, sz = static_cast<int64_t>(nx) * ny;
        const int64_t halo = nz > 1 ? sz : (ny > 1 ? sy : 1);
        const int64_t slice = (c->n + gs::kClusterCTAs - 1) / gs::kClusterCTAs;
        const size_t smem = gs::cluster_smem_bytes(slice, halo);
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        // Measured (tools/cluster_ab.py): C1 (32 K voxels) +39%, C2 (64 K voxels) -5% against the
        // multi-kernel path, whose grid barriers stop dominating as the grid grows.
        cudaFuncAttributes fa{};
        const size_t stat = cudaFuncGetAttributes(&fa, gs::cluster_run_kernel) == cudaSuccess ? fa.sharedSizeBytes : 65536;
        if (c->n <= kClusterMaxVoxels && slice >= halo && slice <= 8 * gs::kSolveThreads &&
            smem + stat + 1024 <= static_cast<size_t>(optin) &&
            cudaFuncSetAttribute(gs::cluster_run_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            raise_cluster_smem(smem)) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(gs::kClusterCTAs);
            cfg.blockDim = dim3(gs::kSolveThreads);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = gs::kClusterCTAs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, gs::cluster_run_kernel, &cfg) == cudaSuccess && clusters > 0) {
                c->cluster_ok = true;
                c->cl_slice = slice;
                c->cl_halo = halo;
                c->cl_smem = smem;
            }
        }
        cudaGetLastError();  // an unsupported attribute only disables the small-grid path
    }
    const size_t vb = sizeof(double) * static_cast<size_t>(c->n);
    for (DevBuf* b : {&c->u, &c->g, &c->f0, &c->f1, &c->t0, &c->t1, &c->out})
        if ((e = b->alloc(vb)) != cudaSuccess) return bail(e, "cudaMalloc(state vectors)");
    if ((e = c->pal.alloc(static_cast<size_t>(c->n))) != cudaSuccess) return bail(e, "cudaMalloc(labels)");
    if ((e = cudaMemsetAsync(c->u.p, 0, vb, c->stream)) != cudaSuccess) return bail(e, "cudaMemset");
    plan_items(c);
    fill_op(c);
    if (build_tensor_maps(c) != GS_OK) {
        g_create_error = c->err;
        gs_destroy(c);
        return GS_ECUDA;
    }
    *out = c;
    return GS_OK;
}

gs_status gs_create_csr(gs_ctx** out, int64_t dim, const int64_t* offs, const int32_t* cols, const double* vals,
                        int device) {
    if (!out || !offs) return fail(nullptr, GS_EINVAL, "gs_create_csr: null argument");
    *out = nullptr;
    // SparseOperator's validation, same messages (sparse.cpp:14-35)
    if (dim < 0) return fail(nullptr, GS_EINVAL, "SparseOperator: negative dimension");
    if (dim == 0) return fail(nullptr, GS_EINVAL, "gs_create_csr: dimension must be >= 1");
    if (dim > INT32_MAX) return fail(nullptr, GS_EINVAL, "gs_create_csr: dimension exceeds int32 column indices");
    if (offs[0] != 0) return fail(nullptr, GS_EINVAL, "SparseOperator: offsets/entries size mismatch");
    const int64_t nnz = offs[dim];
    if (nnz > 0 && (!cols || !vals)) return fail(nullptr, GS_EINVAL, "gs_create_csr: null argument");
    for (int64_t r = 0; r < dim; ++r) {
        if (offs[r] > offs[r + 1]) return fail(nullptr, GS_EINVAL, "SparseOperator: row offsets not monotone");
        for (int64_t q = offs[r]; q < offs[r + 1]; ++q) {
            if (cols[q] < 0 || cols[q] >= dim)
                return fail(nullptr, GS_EINVAL, "SparseOperator: column index out of range");
            if (q > offs[r] && cols[q] <= cols[q - 1])
                return fail(nullptr, GS_EINVAL, "SparseOperator: columns not sorted unique in row " + std::to_string(r));
        }
    }
    gs_ctx* c = nullptr;
    gs_status st = gs_create(&c, static_cast<int>(dim), 1, 1, 1.0, device);
    if (st != GS_OK) return st;
    // transpose for the exact column sums: entries of column k in ascending row order, which is
    // the order the reference's constructor accumulates them (sparse.cpp:36-38)
    std::vector<int64_t> coff(static_cast<size_t>(dim) + 1, 0);
    for (int64_t q = 0; q < nnz; ++q) ++coff[static_cast<size_t>(cols[q]) + 1];
    for (int64_t k = 0; k < dim; ++k) coff[k + 1] += coff[k];
    std::vector<int64_t> fillp(coff.begin(), coff.end() - 1);
    std::vector<double> cabs(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
    for (int64_t r = 0; r < dim; ++r)
        for (int64_t q = offs[r]; q < offs[r + 1]; ++q) cabs[static_cast<size_t>(fillp[cols[q]]++)] = std::fabs(vals[q]);
    auto up = [&](DevBuf& b, const void* src, size_t bytes) -> cudaError_t {
        cudaError_t e = b.alloc(std::max<size_t>(bytes, 8));
        if (e != cudaSuccess) return e;
        return bytes ? cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, c->stream) : cudaSuccess;
    };
    cudaError_t e;
    if ((e = up(c->csr_offs, offs, sizeof(int64_t) * (dim + 1))) != cudaSuccess ||
        (e = up(c->csr_cols, cols, sizeof(int32_t) * nnz)) != cudaSuccess ||
        (e = up(c->csr_vals, vals, sizeof(double) * nnz)) != cudaSuccess ||
        (e = up(c->csc_offs, coff.data(), sizeof(int64_t) * (dim + 1))) != cudaSuccess ||
        (e = up(c->csc_abs, cabs.data(), sizeof(double) * nnz)) != cudaSuccess ||
        (e = cudaStreamSynchronize(c->stream)) != cudaSuccess) {
        g_create_error = std::string("gs_create_csr: ") + cudaGetErrorString(e);
        gs_destroy(c);
        return GS_ECUDA;
    }
    c->is_csr = true;
    c->palette_mode = false;
    st = operator_ready(c);
    if (st != GS_OK) {
        g_create_error = c->err;
        gs_destroy(c);
        return st;
    }
    *out = c;
    return GS_OK;
}

void gs_destroy(gs_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->snap_thread.joinable()) {
        {
            std::lock_guard<std::mutex> lk(c->snap_mu);
            c->snap_stop = true;
        }
        c->snap_cv.notify_all();
        c->snap_thread.join();
    }
    for (SnapSlot& s : c->snap) {
        s.dev.release();
        if (s.ready) cudaEventDestroy(s.ready);
    }
    for (DevBuf* b : {&c->fmt_lens, &c->fmt_offs, &c->fmt_text, &c->fmt_tmp, &c->fmt_tie, &c->fmt_lab, &c->fmt_ltext})
        b->release();
    if (c->host_text) cudaFreeHost(c->host_text);
    if (c->host_u) cudaFreeHost(c->host_u);
    if (c->host_small) cudaFreeHost(c->host_small);
    if (c->snap_stream) cudaStreamDestroy(c->snap_stream);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (DevBuf* b : {&c->csr_offs, &c->csr_cols, &c->csr_vals, &c->csc_offs, &c->csc_abs})
        b->release();
    for (DevBuf* b : {&c->pal, &c->dvox, &c->wtab, &c->dtab, &c->u, &c->g, &c->f0, &c->f1, &c->t0, &c->t1, &c->out,
                      &c->part_b, &c->part_c, &c->part_u, &c->slots, &c->mslots, &c->xchg, &c->x2d, &c->ctrl, &c->metrics, &c->infos,
                      &c->normbits, &c->trace, &c->ens_params, &c->ens_ctl})
        b->release();
    for (cudaEvent_t e : c->events) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ens_events) cudaEventDestroy(e);
    if (c->ens_h2d) cudaStreamDestroy(c->ens_h2d);
    if (c->ens_d2h) cudaStreamDestroy(c->ens_d2h);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* gs_last_error(const gs_ctx* c) {
    if (!c) return g_create_error.c_str();
    return c == t_err_ctx ? t_err.c_str() : c->err.c_str();
}

int64_t gs_num_points(const gs_ctx* c) { return c ? c->n : 0; }

void* gs_stream(gs_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

gs_status gs_set_intensity(gs_ctx* c, const uint8_t* stack, int w, int hgt, int slices, int t_air, int t_white,
                           int t_gray, double d_white, double d_gray) {
    GS_LOCK(c);
    if (c && c->is_csr) return fail(c, GS_EINVAL, "operator is a generic CSR matrix (gs_create_csr)");
    if (!c || !stack) return fail(c, GS_EINVAL, "gs_set_intensity: null argument");
    if (slices < 1 || w < 1 || hgt < 1) return fail(c, GS_EDATA, "resample: degenerate stack");  // imaging.cpp:126-127
    cudaSetDevice(c->device);
    const size_t sb = static_cast<size_t>(w) * hgt * slices;
    DevBuf dstack;
    GS_CUDA(c, dstack.alloc(sb));
    GS_CUDA(c, cudaMemcpyAsync(dstack.p, stack, sb, cudaMemcpyHostToDevice, c->stream));
    const int blocks = static_cast<int>(std::min<int64_t>((c->n + 255) / 256, 148 * 16));
    gs::material_kernel<<<std::max(1, blocks), 256, 0, c->stream>>>(dstack.as<uint8_t>(), w, hgt, slices, c->nx, c->ny,
                                                                    c->nz, t_air, t_white, t_gray, c->pal.as<uint8_t>());
    GS_CUDA(c, cudaGetLastError());
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    dstack.release();
    c->palette_mode = true;
    c->has_labels = true;
    // diffusion_from_materials (imaging.cpp:143-153): Air, Skull -> 0; White, Gray -> d
    gs_status st = upload_palette(c, {0.0, d_white, d_gray, 0.0});
    if (st != GS_OK) return st;
    return operator_ready(c);
}

gs_status gs_set_labels(gs_ctx* c, const uint8_t* labels, double d_white, double d_gray) {
    GS_LOCK(c);
    if (c && c->is_csr) return fail(c, GS_EINVAL, "operator is a generic CSR matrix (gs_create_csr)");
    if (!c || !labels) return fail(c, GS_EINVAL, "gs_set_labels: null argument");
    for (int64_t v = 0; v < c->n; ++v)
        if (labels[v] > 3)
            return fail(c, GS_EDATA, "label volume: byte " + std::to_string(labels[v]) + " is not a material label");
    cudaSetDevice(c->device);
    GS_CUDA(c, cudaMemcpyAsync(c->pal.p, labels, static_cast<size_t>(c->n), cudaMemcpyHostToDevice, c->stream));
    c->palette_mode = true;
    c->has_labels = true;
    gs_status st = upload_palette(c, {0.0, d_white, d_gray, 0.0});
    if (st != GS_OK) return st;
    return operator_ready(c);
}

gs_status gs_set_diffusion(gs_ctx* c, const double* d) {
    GS_LOCK(c);
    if (c && c->is_csr) return fail(c, GS_EINVAL, "operator is a generic CSR matrix (gs_create_csr)");
    if (!c || !d) return fail(c, GS_EINVAL, "gs_set_diffusion: null argument");
    cudaSetDevice(c->device);
    // Palette compression: <= 256 distinct bit patterns -> uint8 index + table (1 B/voxel
    // instead of 8); otherwise the fp64 field is used directly.
    std::vector<uint64_t> keys(static_cast<size_t>(c->n));
    std::memcpy(keys.data(), d, sizeof(double) * keys.size());
    std::vector<uint64_t> uniq(keys);
    uniq.push_back(0);  // palette index 0 is always D = +0.0: TMA zero-fill outside the grid reads it
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    c->has_labels = false;
    if (uniq.size() <= 256) {
        std::vector<uint8_t> idx(keys.size());
        for (size_t v = 0; v < keys.size(); ++v)
            idx[v] = static_cast<uint8_t>(std::lower_bound(uniq.begin(), uniq.end(), keys[v]) - uniq.begin());
        std::vector<double> dvals(uniq.size());
        std::memcpy(dvals.data(), uniq.data(), sizeof(double) * uniq.size());
        GS_CUDA(c, cudaMemcpyAsync(c->pal.p, idx.data(), idx.size(), cudaMemcpyHostToDevice, c->stream));
        GS_CUDA(c, cudaStreamSynchronize(c->stream));
        c->palette_mode = true;
        gs_status st = upload_palette(c, dvals);
        if (st != GS_OK) return st;
    } else {
        GS_CUDA(c, c->dvox.alloc(sizeof(double) * static_cast<size_t>(c->n)));
        GS_CUDA(c, cudaMemcpyAsync(c->dvox.p, d, sizeof(double) * static_cast<size_t>(c->n), cudaMemcpyHostToDevice,
                                   c->stream));
        GS_CUDA(c, c->wtab.alloc(256 * sizeof(double)));
        GS_CUDA(c, cudaStreamSynchronize(c->stream));
        c->palette_mode = false;
    }
    return operator_ready(c);
}

gs_status gs_get_labels(gs_ctx* c, uint8_t* labels) {
    GS_LOCK(c);
    if (!c || !labels) return fail(c, GS_EINVAL, "gs_get_labels: null argument");
    if (!c->has_labels) return fail(c, GS_EINVAL, "gs_get_labels: operator was not built from material labels");
    cudaSetDevice(c->device);
    GS_CUDA(c, cudaMemcpyAsync(labels, c->pal.p, static_cast<size_t>(c->n), cudaMemcpyDeviceToHost, c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    return GS_OK;
}

gs_status gs_get_diffusion(gs_ctx* c, double* d) {
    GS_LOCK(c);
    if (!c || !d) return fail(c, GS_EINVAL, "gs_get_diffusion: null argument");
    gs_status st = ensure_operator(c);
    if (st != GS_OK) return st;
    cudaSetDevice(c->device);
    const size_t bytes = sizeof(double) * static_cast<size_t>(c->n);
    if (c->palette_mode) {
        const int blocks = static_cast<int>(std::min<int64_t>((c->n + 255) / 256, 148 * 16));
        gs::expand_palette_kernel<<<std::max(1, blocks), 256, 0, c->stream>>>(c->pal.as<uint8_t>(), c->dtab.as<double>(),
                                                                               c->n, c->out.as<double>());
        GS_CUDA(c, cudaGetLastError());
        GS_CUDA(c, cudaMemcpyAsync(d, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    } else {
        GS_CUDA(c, cudaMemcpyAsync(d, c->dvox.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    return GS_OK;
}

gs_status gs_one_norm(gs_ctx* c, double* out) {
    GS_LOCK(c);
    if (!c || !out) return fail(c, GS_EINVAL, "gs_one_norm: null argument");
    gs_status st = ensure_operator(c);
    if (st != GS_OK) return st;
    *out = c->anorm;
    return GS_OK;
}

gs_status gs_apply(gs_ctx* c, const double* x, double* y) {
    GS_LOCK(c);
    if (!c || !x || !y) return fail(c, GS_EINVAL, "gs_apply: null argument");
    gs_status st = ensure_operator(c);
    if (st != GS_OK) return st;
    cudaSetDevice(c->device);
    const size_t bytes = sizeof(double) * static_cast<size_t>(c->n);
    GS_CUDA(c, cudaMemcpyAsync(c->g.p, x, bytes, cudaMemcpyHostToDevice, c->stream));
    gs::SolveParams p{};
    p.mode = gs::kModeApply;
    p.n_steps = 1;
    st = launch_solve(c, p, 1, nullptr, nullptr);
    if (st != GS_OK) return st;
    GS_CUDA(c, cudaMemcpyAsync(y, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    return GS_OK;
}

gs_status gs_set_state(gs_ctx* c, const double* u) {
    GS_LOCK(c);
    if (!c || !u) return fail(c, GS_EINVAL, "gs_set_state: null argument");
    cudaSetDevice(c->device);
    GS_CUDA(c, cudaMemcpyAsync(c->u.p, u, sizeof(double) * static_cast<size_t>(c->n), cudaMemcpyHostToDevice,
                               c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    return GS_OK;
}

gs_status gs_get_state(gs_ctx* c, double* u) {
    GS_LOCK(c);
    if (!c || !u) return fail(c, GS_EINVAL, "gs_get_state: null argument");
    cudaSetDevice(c->device);
    GS_CUDA(c, cudaMemcpyAsync(u, c->u.p, sizeof(double) * static_cast<size_t>(c->n), cudaMemcpyDeviceToHost,
                               c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    return GS_OK;
}

double* gs_state_device_ptr(gs_ctx* c) { return c ? c->u.as<double>() : nullptr; }

gs_status gs_select_params(double norm_tA, double tol, int* s, int* m) {
    if (!s || !m) return GS_EINVAL;
    if (!std::isfinite(norm_tA) || norm_tA < 0.0) {
        g_create_error = "select_params: operator norm must be finite and nonnegative";
        return GS_EINVAL;
    }
    if (!tol_ok(tol)) {
        g_create_error = "select_params: tolerance must lie in (0, 1)";
        return GS_EINVAL;
    }
    double rtab[gs::kMaxDegree + 1];
    fill_rtab(tol, rtab);
    *s = 1;
    *m = 1;
    if (norm_tA == 0.0) return GS_OK;
    double best_cost = -1.0;
    for (int mm = 1; mm <= gs::kMaxDegree; ++mm) {
        const double c = std::ceil(norm_tA / rtab[mm]);
        const double stages = (1.0 < c) ? c : 1.0;
        if (stages > 2e9) continue;
        const double cost = stages * mm;
        if (best_cost < 0.0 || cost < best_cost) {
            best_cost = cost;
            *s = static_cast<int>(stages);
            *m = mm;
        }
    }
    if (best_cost < 0.0) {
        g_create_error = "select_params: scaled operator norm too large for any stage count";
        return GS_ENUMERIC;
    }
    return GS_OK;
}

static gs_status action(gs_ctx* c, int mode, double t, const double* b, double tol, double* out,
                        gs_step_info* info) {
    GS_LOCK(c);
    const char* who = mode == gs::kModeExpmv ? "expmv" : "phi1v";
    if (!c || !b || !out) return fail(c, GS_EINVAL, std::string(who) + ": null argument");
    if (!tol_ok(tol)) return fail(c, GS_EINVAL, std::string(who) + ": tolerance must lie in (0, 1)");
    gs_status st = ensure_operator(c);
    if (st != GS_OK) return st;
    const size_t bytes = sizeof(double) * static_cast<size_t>(c->n);
    if (t == 0.0) {  // expact.cpp:69, :108
        std::memcpy(out, b, bytes);
        if (info) {
            std::memset(info, 0, sizeof *info);
            info->s = info->m = 1;
            info->branch = 1;
        }
        return GS_OK;
    }
    cudaSetDevice(c->device);
    GS_CUDA(c, cudaMemcpyAsync(c->g.p, b, bytes, cudaMemcpyHostToDevice, c->stream));
    gs::SolveParams p{};
    p.mode = mode;
    p.n_steps = 1;
    p.tau = t;
    p.tol = tol;
    fill_rtab(tol, p.rtab);
    st = launch_solve(c, p, 1, nullptr, info);
    if (st != GS_OK) return st;
    GS_CUDA(c, cudaMemcpyAsync(out, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    return GS_OK;
}

gs_status gs_expmv(gs_ctx* c, double t, const double* b, double tol, double* out, gs_step_info* info) {
    return action(c, gs::kModeExpmv, t, b, tol, out, info);
}

gs_status gs_phi1v(gs_ctx* c, double t, const double* b, double tol, double* out, gs_step_info* info) {
    return action(c, gs::kModePhi1v, t, b, tol, out, info);
}

gs_status gs_run(gs_ctx* c, int n_steps, double rho, double tau, double tol, const double origin[3],
                 const double seed_center[3], double front_threshold, gs_metrics* metrics, gs_step_info* infos) {
    GS_LOCK(c);
    if (!c) return fail(c, GS_EINVAL, "run: null context");
    if (n_steps < 0) return fail(c, GS_EINVAL, "run: negative step count");
    if (!tol_ok(tol)) return fail(c, GS_EINVAL, "phi1v: tolerance must lie in (0, 1)");
    gs_status st = ensure_operator(c);
    if (st != GS_OK) return st;
    if (metrics && (!origin || !seed_center)) return fail(c, GS_EINVAL, "run: metrics need origin and seed center");
    cudaSetDevice(c->device);
    gs::SolveParams p{};
    p.mode = gs::kModeRun;
    p.n_steps = n_steps;
    p.rho = rho;
    p.tau = tau;
    p.tol = tol;
    p.h = c->h;
    p.front_threshold = front_threshold;
    for (int a = 0; a < 3; ++a) {
        p.origin[a] = origin ? origin[a] : 0.0;
        p.center[a] = seed_center ? seed_center[a] : 0.0;
    }
    fill_rtab(tol, p.rtab);
    return launch_solve(c, p, n_steps, reinterpret_cast<gs_metrics*>(metrics), infos);
}

namespace {

// gs_run_ensemble / gs_step_ensemble_host: the members' SolveParams and launch geometry.
struct EnsPlan {
    std::vector<gs::SolveParams> P;
    int groups = 1, grp = 1, sb = 1, fuse = 2;
    int num_sms = 1;
    int sq = 1;   // CTAs per member of the seqsum item pass
    int sq1 = 1;  // ... and of its tile pass
    bool batched = false;
    bool seq_exact = true;  // the members' SolveParams::seq_exact (one environment, one value)
};

// Validate the members and, when they can take the batched path, set up every member's
// scratch and SolveParams (errors on ctxs[0], naming the member).
gs_status ens_prepare(gs_ctx* const* ctxs, int n_members, int n_steps, const double* rhos, double tau, double tol,
                      const double* origins, const double* centers, double front_threshold, gs_metrics* metrics,
                      gs_step_info* infos, int groups, EnsPlan& plan) {
    if (!ctxs || n_members < 1 || !rhos) return fail(nullptr, GS_EINVAL, "run_ensemble: null argument or no members");
    for (int i = 0; i < n_members; ++i) {
        if (!ctxs[i]) return fail(nullptr, GS_EINVAL, "run_ensemble: null member context");
        for (int j = 0; j < i; ++j)  // a member's buffers must belong to it alone
            if (ctxs[j] == ctxs[i]) return fail(ctxs[i], GS_EINVAL, "run_ensemble: a context appears twice");
    }
    gs_ctx* const c0 = ctxs[0];
    if (n_steps < 0) return fail(c0, GS_EINVAL, "run: negative step count");
    if (!tol_ok(tol)) return fail(c0, GS_EINVAL, "phi1v: tolerance must lie in (0, 1)");
    if (metrics && (!origins || !centers)) return fail(c0, GS_EINVAL, "run: metrics need origin and seed center");
    bool batched = std::getenv("GS_ENS_SEQUENTIAL") == nullptr && std::getenv("GS_DISABLE_TMA") == nullptr;
    int thin = 0;
    for (int i = 0; i < n_members; ++i) {
        gs_ctx* c = ctxs[i];
        const gs_status st = ensure_operator(c);
        if (st != GS_OK) return fail(c0, st, "run_ensemble: member " + std::to_string(i) + ": " + c->err);
        if (c->device != c0->device) return fail(c0, GS_EINVAL, "run_ensemble: members on different devices");
        batched = batched && c->tma_ok && c->palette_mode && !c->is_csr;
        thin += c->nz < 8;
    }
    plan.batched = batched && (thin == 0 || thin == n_members);  // one Taylor instantiation per launch
    if (!plan.batched) return GS_OK;
    cudaSetDevice(c0->device);
    // CTA groups of the Taylor launch: each runs one member at a time on num_sms / groups SMs
    if (groups <= 0) {
        groups = kEnsembleGroups;
        if (const char* e = std::getenv("GS_ENS_GROUPS")) groups = std::atoi(e);
    }
    plan.groups = std::max(1, std::min({groups, n_members, c0->num_sms}));
    plan.grp = c0->num_sms / plan.groups;
    plan.num_sms = c0->capacity > 0 ? std::min(c0->num_sms, c0->capacity) : c0->num_sms;
    plan.sb = 1;
    for (int i = 0; i < n_members; ++i) plan.sb = std::max(plan.sb, stream_blocks(ctxs[i]));
    plan.fuse = thin ? 4 : 2;
    plan.seq_exact = std::getenv("GS_TREE_SUMS") == nullptr;
    {
        int tiles = 1;
        for (int i = 0; i < n_members; ++i)
            tiles = std::max(tiles, static_cast<int>((ctxs[i]->n + gs::kSeqTileElems - 1) / gs::kSeqTileElems));
        plan.sq = seq_ctas(c0, tiles, n_members);
        plan.sq1 = std::max(1, std::min(tiles, 2 * c0->num_sms / n_members));
        if (const char* e = std::getenv("GS_SEQ_CTAS1")) plan.sq1 = std::max(1, std::min(tiles, std::atoi(e)));
    }
    plan.P.assign(static_cast<size_t>(n_members), gs::SolveParams{});
    for (int i = 0; i < n_members; ++i) {
        gs_ctx* c = ctxs[i];
        gs::SolveParams& p = plan.P[i];
        p.mode = gs::kModeRun;
        p.n_steps = n_steps;
        p.rho = rhos[i];
        p.tau = tau;
        p.tol = tol;
        p.h = c->h;
        p.front_threshold = front_threshold;
        for (int a = 0; a < 3; ++a) {
            p.origin[a] = origins ? origins[3 * i + a] : 0.0;
            p.center[a] = centers ? centers[3 * i + a] : 0.0;
        }
        fill_rtab(tol, p.rtab);
        gs_status st = setup_solve(c, p, plan.grp, plan.sb, n_steps, metrics, infos);
        if (st == GS_OK) st = c->stream && cudaStreamSynchronize(c->stream) != cudaSuccess ? GS_ECUDA : GS_OK;
        if (st != GS_OK)
            return fail(c0, st, "run_ensemble: member " + std::to_string(i) + ": " + (c->err.empty() ? "CUDA error" : c->err));
    }
    return GS_OK;
}

// n_steps batched steps of the n members whose SolveParams start at dP, on stream st; ctl
// holds ens_ctl_words(groups) + n words.
// tc (optional): a context with kernel timing on -- CUDA events bracket each step's Taylor
// launch on st (gs_get_kernel_times of that context then reports them under "taylor").
cudaError_t ens_launch(const EnsPlan& plan, const gs::SolveParams* dP, int n, int n_steps, bool metrics,
                       unsigned* ctl, cudaStream_t st, gs_ctx* tc = nullptr) {
    if (tc && !tc->ktime) tc = nullptr;
    if (tc)
        while (tc->events.size() < 2 * static_cast<size_t>(n_steps)) {
            cudaEvent_t ev;
            const cudaError_t r = cudaEventCreate(&ev);
            if (r != cudaSuccess) return r;
            tc->events.push_back(ev);
        }
    const int groups = std::min(plan.groups, n), grp = plan.grp, sb = plan.sb;
    const unsigned* order = ctl + gs::ens_ctl_words(groups);
    const dim3 blk(gs::kSolveThreads);
    cudaError_t e = cudaSuccess;
    if (metrics) {
        gs::ens_metrics_kernel<<<n * sb, blk, 0, st>>>(dP, sb);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    for (int step = 0; step < n_steps; ++step) {
        gs::ens_prep_kernel<<<n * grp, blk, gs::kRingBytes, st>>>(dP, grp, step);
        if (plan.seq_exact) {
            gs::ens_seqsum_tiles_kernel<<<n * plan.sq1, blk, 0, st>>>(dP, plan.sq1, 0);
            gs::ens_seqsum_items_kernel<<<n * plan.sq, blk, 0, st>>>(dP, plan.sq, 0);
        }
        gs::ens_border_kernel<<<n * sb, blk, 0, st>>>(dP, sb, grp, step);
        if (plan.seq_exact) {
            gs::ens_seqsum_tiles_kernel<<<n * plan.sq1, blk, 0, st>>>(dP, plan.sq1, 1);
            gs::ens_seqsum_items_kernel<<<n * plan.sq, blk, 0, st>>>(dP, plan.sq, 1);
        }
        gs::ens_order_kernel<<<1, 256, 0, st>>>(dP, n, ctl + gs::ens_ctl_words(groups));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(ctl, 0, sizeof(unsigned) * gs::ens_ctl_words(groups), st)) != cudaSuccess) return e;
        // the SMs left over by groups * grp go one each to the first groups
        // (measured on C5: 2150 member-steps/s with the extra CTAs against 2156 without -- the
        // longer groups finish no sooner -- so GS_ENS_EXTRA=1 opts in, for A/B)
        int nm = n, g = grp, bb = sb, sp = step, extra = std::max(0, std::min(groups, plan.num_sms - groups * grp));
        if (!std::getenv("GS_ENS_EXTRA")) extra = 0;
        void* args[] = {const_cast<gs::SolveParams**>(&dP), &nm, &g, &bb, &sp, &ctl, const_cast<unsigned**>(&order),
                        &extra};
        if (tc && (e = cudaEventRecord(tc->events[2 * step], st)) != cudaSuccess) return e;
        if ((e = cudaLaunchCooperativeKernel(gs::ens_taylor_kernel_fn(plan.fuse), dim3(groups * grp + extra), blk, args,
                                             gs::kDynSmemBytes, st)) != cudaSuccess)
            return e;
        if (tc && (e = cudaEventRecord(tc->events[2 * step + 1], st)) != cudaSuccess) return e;
        gs::ens_update_kernel<<<n * sb, blk, 0, st>>>(dP, sb, step);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return e;
}

// Per-member status after a batched run: the first failure, reported on ctxs[0].
gs_status ens_status(gs_ctx* const* ctxs, int n_members, const std::vector<gs::Ctrl>& ctrl) {
    for (int i = 0; i < n_members; ++i) {
        if (ctrl[i].status == GS_OK) continue;
        const std::string who = "run_ensemble: member " + std::to_string(i) + ": ";
        if (ctrl[i].detail == 2)
            return fail(ctxs[0], GS_ENUMERIC, who + "expmv: series diverged to non-finite values; reduce t");
        if (ctrl[i].status == GS_EINVAL)
            return fail(ctxs[0], GS_EINVAL, who + "select_params: operator norm must be finite and nonnegative");
        return fail(ctxs[0], GS_ENUMERIC, who + "select_params: scaled operator norm too large for any stage count");
    }
    return GS_OK;
}

}  // namespace

gs_status gs_run_ensemble(gs_ctx* const* ctxs, int n_members, int n_steps, const double* rhos, double tau, double tol,
                          const double* origins, const double* centers, double front_threshold, gs_metrics* metrics,
                          gs_step_info* infos, int groups) {
    MultiLock lk(ctxs, n_members);
    EnsPlan plan;
    gs_status st0 = ens_prepare(ctxs, n_members, n_steps, rhos, tau, tol, origins, centers, front_threshold, metrics,
                                infos, groups, plan);
    if (st0 != GS_OK) return st0;
    if (!plan.batched) {
        // members the batched path cannot take run one after another, each on the whole GPU
        for (int i = 0; i < n_members; ++i) {
            const gs_status st = gs_run(ctxs[i], n_steps, rhos[i], tau, tol, origins ? origins + 3 * i : nullptr,
                                        centers ? centers + 3 * i : nullptr, front_threshold,
                                        metrics ? metrics + static_cast<size_t>(i) * (n_steps + 1) : nullptr,
                                        infos ? infos + static_cast<size_t>(i) * n_steps : nullptr);
            if (st != GS_OK) return st;
        }
        return GS_OK;
    }
    gs_ctx* const c0 = ctxs[0];
    GS_CUDA(c0, c0->ens_params.alloc(sizeof(gs::SolveParams) * static_cast<size_t>(n_members)));
    GS_CUDA(c0, c0->ens_ctl.alloc(sizeof(unsigned) * (gs::ens_ctl_words(plan.groups) + n_members)));
    GS_CUDA(c0, cudaMemcpyAsync(c0->ens_params.p, plan.P.data(), sizeof(gs::SolveParams) * static_cast<size_t>(n_members),
                                cudaMemcpyHostToDevice, c0->stream));
    cudaStream_t st = c0->stream;
    GS_CUDA(c0, ens_launch(plan, c0->ens_params.as<gs::SolveParams>(), n_members, n_steps, metrics != nullptr,
                           c0->ens_ctl.as<unsigned>(), st, c0));
    std::vector<gs::Ctrl> ctrl(static_cast<size_t>(n_members));
    for (int i = 0; i < n_members; ++i) {
        gs_ctx* c = ctxs[i];
        GS_CUDA(c0, cudaMemcpyAsync(&ctrl[i], c->ctrl.p, sizeof(gs::Ctrl), cudaMemcpyDeviceToHost, st));
        if (metrics)
            GS_CUDA(c0, cudaMemcpyAsync(metrics + static_cast<size_t>(i) * (n_steps + 1), c->metrics.p,
                                        sizeof(double) * 4 * (n_steps + 1), cudaMemcpyDeviceToHost, st));
        if (infos && n_steps > 0)
            GS_CUDA(c0, cudaMemcpyAsync(infos + static_cast<size_t>(i) * n_steps, c->infos.p,
                                        sizeof(gs_step_info) * n_steps, cudaMemcpyDeviceToHost, st));
    }
    GS_CUDA(c0, cudaStreamSynchronize(st));
    if (c0->ktime) {  // the batched Taylor launches of this call (kind 2 = taylor, as gs_run reports it)
        for (int k = 0; k < 4; ++k) {
            c0->kms[k] = 0.0;
            c0->kcount[k] = 0;
        }
        for (int q = 0; q < n_steps; ++q) {
            float ms = 0.f;
            GS_CUDA(c0, cudaEventElapsedTime(&ms, c0->events[2 * q], c0->events[2 * q + 1]));
            c0->kms[2] += ms;
            c0->kcount[2] += 1;
        }
    }
    return ens_status(ctxs, n_members, ctrl);
}

gs_status gs_step_ensemble_host(gs_ctx* const* ctxs, int n_members, const double* const* u_in, double* const* u_out,
                                const double* rhos, double tau, double tol, gs_step_info* infos, int groups,
                                int chunks) {
    MultiLock lk(ctxs, n_members);
    if (!u_in || !u_out) return fail(ctxs ? ctxs[0] : nullptr, GS_EINVAL, "step_ensemble: null argument");
    for (int i = 0; ctxs && i < n_members; ++i)
        if (!u_in[i] || !u_out[i]) return fail(ctxs[0], GS_EINVAL, "step_ensemble: null member vector");
    EnsPlan plan;
    // value semantics: every member steps its staging (`out`) buffer, its resident u untouched
    for (int i = 0; ctxs && i < n_members; ++i)
        if (ctxs[i]) ctxs[i]->stage_swap = true;
    gs_status st0 = ens_prepare(ctxs, n_members, 1, rhos, tau, tol, nullptr, nullptr, 0.1, nullptr, infos, groups, plan);
    for (int i = 0; ctxs && i < n_members; ++i)
        if (ctxs[i]) ctxs[i]->stage_swap = false;
    if (st0 != GS_OK) return st0;
    if (!plan.batched) {
        for (int i = 0; i < n_members; ++i) {
            const gs_status st = gs_step_host(ctxs[i], u_in[i], rhos[i], tau, tol, u_out[i], infos ? infos + i : nullptr);
            if (st != GS_OK) return st;
        }
        return GS_OK;
    }
    gs_ctx* const c0 = ctxs[0];
    if (chunks <= 0) chunks = kEnsembleChunks;
    chunks = std::max(1, std::min(chunks, n_members));
    // H2D, compute and D2H on three streams: chunk k's copies overlap chunk k-1's and k+1's
    // steps (pinned host vectors make the copies asynchronous)
    if (!c0->ens_h2d) GS_CUDA(c0, cudaStreamCreateWithFlags(&c0->ens_h2d, cudaStreamNonBlocking));
    if (!c0->ens_d2h) GS_CUDA(c0, cudaStreamCreateWithFlags(&c0->ens_d2h, cudaStreamNonBlocking));
    while (static_cast<int>(c0->ens_events.size()) < 2 * chunks) {
        cudaEvent_t e;
        GS_CUDA(c0, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c0->ens_events.push_back(e);
    }
    GS_CUDA(c0, c0->ens_params.alloc(sizeof(gs::SolveParams) * static_cast<size_t>(n_members)));
    GS_CUDA(c0, c0->ens_ctl.alloc(sizeof(unsigned) * (gs::ens_ctl_words(plan.groups) + n_members)));
    GS_CUDA(c0, cudaMemcpyAsync(c0->ens_params.p, plan.P.data(), sizeof(gs::SolveParams) * static_cast<size_t>(n_members),
                                cudaMemcpyHostToDevice, c0->stream));
    const gs::SolveParams* dP = c0->ens_params.as<gs::SolveParams>();
    const size_t bytes = sizeof(double);
    for (int k = 0; k < chunks; ++k) {
        const int lo = k * n_members / chunks, hi = (k + 1) * n_members / chunks;
        for (int i = lo; i < hi; ++i)
            GS_CUDA(c0, cudaMemcpyAsync(ctxs[i]->out.p, u_in[i], bytes * static_cast<size_t>(ctxs[i]->n),
                                        cudaMemcpyHostToDevice, c0->ens_h2d));
        GS_CUDA(c0, cudaEventRecord(c0->ens_events[2 * k], c0->ens_h2d));
        GS_CUDA(c0, cudaStreamWaitEvent(c0->stream, c0->ens_events[2 * k], 0));
        GS_CUDA(c0, ens_launch(plan, dP + lo, hi - lo, 1, false, c0->ens_ctl.as<unsigned>(), c0->stream));
        GS_CUDA(c0, cudaEventRecord(c0->ens_events[2 * k + 1], c0->stream));
        GS_CUDA(c0, cudaStreamWaitEvent(c0->ens_d2h, c0->ens_events[2 * k + 1], 0));
        for (int i = lo; i < hi; ++i)
            GS_CUDA(c0, cudaMemcpyAsync(u_out[i], ctxs[i]->out.p, bytes * static_cast<size_t>(ctxs[i]->n),
                                        cudaMemcpyDeviceToHost, c0->ens_d2h));
    }
    std::vector<gs::Ctrl> ctrl(static_cast<size_t>(n_members));
    for (int i = 0; i < n_members; ++i) {
        GS_CUDA(c0, cudaMemcpyAsync(&ctrl[i], ctxs[i]->ctrl.p, sizeof(gs::Ctrl), cudaMemcpyDeviceToHost, c0->ens_d2h));
        if (infos)
            GS_CUDA(c0, cudaMemcpyAsync(infos + i, ctxs[i]->infos.p, sizeof(gs_step_info), cudaMemcpyDeviceToHost,
                                        c0->ens_d2h));
    }
    GS_CUDA(c0, cudaStreamSynchronize(c0->ens_d2h));
    GS_CUDA(c0, cudaStreamSynchronize(c0->stream));
    return ens_status(ctxs, n_members, ctrl);
}

gs_status gs_step(gs_ctx* c, double rho, double tau, double tol, gs_step_info* info) {
    return gs_run(c, 1, rho, tau, tol, nullptr, nullptr, 0.1, nullptr, info);
}

gs_status gs_step_host(gs_ctx* c, const double* u, double rho, double tau, double tol, double* out,
                       gs_step_info* info) {
    if (!c || !u || !out) return fail(c, GS_EINVAL, "gs_step_host: null argument");
    // u in, one step, u' out on the context's stream with a single synchronisation
    GS_LOCK(c);
    c->stage_in = u;
    c->stage_out = out;
    c->stage_swap = true;
    const gs_status st = gs_step(c, rho, tau, tol, info);
    c->stage_in = nullptr;
    c->stage_out = nullptr;
    c->stage_swap = false;
    return st;
}

gs_status gs_seed_initial(gs_ctx* c, const double origin[3], double amplitude, double width, const double center[3],
                          int mask, double* u) {
    GS_LOCK(c);
    if (!c || !u || !center) return fail(c, GS_EINVAL, "seed_initial: null argument");
    const double o[3] = {origin ? origin[0] : 0.0, origin ? origin[1] : 0.0, origin ? origin[2] : 0.0};
    // Grid::contains (grid.hpp:43-50)
    const int dims[3] = {c->nx, c->ny, c->nz};
    for (int a = 0; a < 3; ++a) {
        const double lo = o[a], hi = o[a] + (dims[a] - 1) * c->h;
        if (center[a] < lo || center[a] > hi)
            return fail(c, GS_EDATA, "seed center lies outside the computational domain");
    }
    // the D == 0 mask (seed_initial(d, cfg), integrator.cpp:44-48): palette indices + table
    // (1 byte per voxel back from the device), or the fp64 field
    std::vector<uint8_t> pal;
    std::vector<double> d;
    if (mask) {
        gs_status st = ensure_operator(c);
        if (st != GS_OK) return st;
        if (c->palette_mode && !c->is_csr) {
            pal.resize(static_cast<size_t>(c->n));
            GS_CUDA(c, cudaMemcpyAsync(pal.data(), c->pal.p, pal.size(), cudaMemcpyDeviceToHost, c->stream));
            GS_CUDA(c, cudaStreamSynchronize(c->stream));
        } else {
            d.resize(static_cast<size_t>(c->n));
            st = gs_get_diffusion(c, d.data());
            if (st != GS_OK) return st;
        }
    }
    auto dead = [&](int64_t v) {
        return pal.empty() ? d[static_cast<size_t>(v)] == 0.0 : c->dtab_host[pal[static_cast<size_t>(v)]] == 0.0;
    };
    // integrator.cpp:32-50; sq_dist integrator.cpp:23-29 (this file is built with
    // -ffp-contract=off on the host side too).  Planes are split over host threads: every
    // voxel is computed independently with the same glibc exp, so the result does not
    // depend on the split.
    const int nthreads = static_cast<int>(std::min<int64_t>(std::max(1, gsio::default_threads()), c->nz));
    auto planes = [&](int k0, int k1) {
        for (int k = k0 + 1; k <= k1; ++k) {
            int64_t v = static_cast<int64_t>(k - 1) * c->nx * c->ny;
            for (int j = 1; j <= c->ny; ++j)
                for (int i = 1; i <= c->nx; ++i, ++v) {
                    const double px = o[0] + (i - 1) * c->h, py = o[1] + (j - 1) * c->h, pz = o[2] + (k - 1) * c->h;
                    const double dx = px - center[0], dy = py - center[1], dz = pz - center[2];
                    const double sq = dx * dx + dy * dy + dz * dz;
                    u[v] = amplitude * std::exp(-width * sq);
                    if (mask && dead(v)) u[v] = 0.0;
                }
        }
    };
    if (nthreads <= 1 || c->n < (1 << 16)) {
        planes(0, c->nz);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t)
            pool.emplace_back(planes, static_cast<int>(static_cast<int64_t>(c->nz) * t / nthreads),
                              static_cast<int>(static_cast<int64_t>(c->nz) * (t + 1) / nthreads));
        for (auto& th : pool) th.join();
    }
    return GS_OK;
}

gs_status gs_set_kernel_timing(gs_ctx* c, int enable) {
    GS_LOCK(c);
    if (!c) return fail(c, GS_EINVAL, "gs_set_kernel_timing: null context");
    c->ktime = enable != 0;
    return GS_OK;
}

gs_status gs_get_kernel_times(gs_ctx* c, double ms[4], int launches[4]) {
    GS_LOCK(c);
    if (!c || !ms || !launches) return fail(c, GS_EINVAL, "gs_get_kernel_times: null argument");
    for (int k = 0; k < 4; ++k) {
        ms[k] = c->kms[k];
        launches[k] = c->kcount[k];
    }
    return GS_OK;
}

gs_status gs_set_trace(gs_ctx* c, int capacity) {
    GS_LOCK(c);
    if (!c || capacity < 0) return fail(c, GS_EINVAL, "gs_set_trace: bad argument");
    c->trace_cap = capacity;
    return GS_OK;
}

gs_status gs_get_trace(gs_ctx* c, uint64_t* pairs, int capacity, int* count) {
    GS_LOCK(c);
    if (!c || !pairs || !count) return fail(c, GS_EINVAL, "gs_get_trace: null argument");
    int n = 0;
    const int have = static_cast<int>(c->trace_host.size() / 2);
    while (n < have && n < capacity && c->trace_host[2 * n] != 0) {
        pairs[2 * n] = c->trace_host[2 * n];
        pairs[2 * n + 1] = c->trace_host[2 * n + 1];
        ++n;
    }
    *count = n;
    return GS_OK;
}

gs_status gs_snapshot_vtk(gs_ctx* c, const char* path, const double origin[3], const uint8_t* labels) {
    GS_LOCK(c);
    if (!c || !path || !origin) return fail(c, GS_EINVAL, "gs_snapshot_vtk: null argument");
    cudaSetDevice(c->device);
    // open now so an unwritable path fails at this snapshot, as write_vtk does (vtk.cpp:66-68)
    std::FILE* f = std::fopen(path, "w");
    if (!f) return fail(c, GS_EDATA, std::string("cannot open ") + path + " for writing");
    int slot = -1;
    {
        std::unique_lock<std::mutex> lk(c->snap_mu);
        c->snap_cv.wait(lk, [&] {
            if (c->snap_code != GS_OK) return true;
            for (int s = 0; s < kSnapSlots; ++s)
                if (!c->snap[s].busy) return true;
            return false;
        });
        if (c->snap_code != GS_OK) {  // an earlier snapshot failed: report it here
            std::fclose(f);
            const gs_status code = c->snap_code;
            c->snap_code = GS_OK;
            return fail(c, code, c->snap_err);
        }
        for (int s = 0; s < kSnapSlots && slot < 0; ++s)
            if (!c->snap[s].busy) slot = s;
        c->snap[slot].busy = true;
    }
    SnapSlot& sl = c->snap[slot];
    const size_t bytes = sizeof(double) * static_cast<size_t>(c->n);
    auto release = [&](cudaError_t e, const char* where) {
        std::fclose(f);
        {
            std::lock_guard<std::mutex> lk(c->snap_mu);
            sl.busy = false;
        }
        return cuda_fail(c, e, where);
    };
    cudaError_t e = sl.dev.alloc(bytes);
    if (e == cudaSuccess && !sl.ready) e = cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming);
    if (e != cudaSuccess) return release(e, "gs_snapshot_vtk: allocation");
    // device copy on the compute stream (the next step overwrites u); the writer thread
    // formats it on the GPU and brings the text back on its own stream
    e = cudaMemcpyAsync(sl.dev.p, c->u.p, bytes, cudaMemcpyDeviceToDevice, c->stream);
    if (e == cudaSuccess) e = cudaEventRecord(sl.ready, c->stream);
    if (e != cudaSuccess) return release(e, "gs_snapshot_vtk: copy");

    SnapJob job;
    job.slot = slot;
    job.f = f;
    job.path = path;
    std::copy(origin, origin + 3, job.origin);
    if (labels) job.labels.assign(labels, labels + c->n);
    {
        std::lock_guard<std::mutex> lk(c->snap_mu);
        c->snap_q.push_back(std::move(job));
        if (!c->snap_thread.joinable()) c->snap_thread = std::thread([c] { snapshot_writer(c); });
    }
    c->snap_cv.notify_all();
    return GS_OK;
}

int gs_uses_cluster(const gs_ctx* c) {
    return (c && c->cluster_ok && c->palette_mode && !c->is_csr && std::getenv("GS_NO_CLUSTER") == nullptr) ? 1 : 0;
}

int gs_uses_flat2d(const gs_ctx* c) {
    if (!c || c->nz != 1 || !c->palette_mode || c->is_csr || !gs::taylor2d_kernel_fn()) return 0;
    const int t2d = tiles_2d(c);
    return (t2d <= c->cap2d && std::getenv("GS_NO_2D") == nullptr) ? 1 : 0;
}

gs_status gs_snapshot_flush(gs_ctx* c) {
    if (!c) return fail(c, GS_EINVAL, "gs_snapshot_flush: null argument");
    std::unique_lock<std::mutex> lk(c->snap_mu);
    c->snap_cv.wait(lk, [&] {
        if (!c->snap_q.empty()) return false;
        for (const SnapSlot& s : c->snap)
            if (s.busy) return false;
        return true;
    });
    if (c->snap_code != GS_OK) {
        const gs_status code = c->snap_code;
        c->snap_code = GS_OK;
        c->err = c->snap_err;
        return code;
    }
    return GS_OK;
}

gs_status gs_matter_fractions(gs_ctx* c, double* white, double* gray) {
    GS_LOCK(c);
    if (!c || !white || !gray) return fail(c, GS_EINVAL, "gs_matter_fractions: null argument");
    if (!c->has_labels) return fail(c, GS_EINVAL, "gs_matter_fractions: operator was not built from material labels");
    cudaSetDevice(c->device);
    DevBuf cnt;
    GS_CUDA(c, cnt.alloc(4 * sizeof(unsigned long long)));
    GS_CUDA(c, cudaMemsetAsync(cnt.p, 0, 4 * sizeof(unsigned long long), c->stream));
    const int blocks = std::max(1, static_cast<int>(std::min<int64_t>((c->n / 16 + 255) / 256, c->num_sms * 8)));
    gs::label_count_kernel<<<blocks, 256, 0, c->stream>>>(c->pal.as<uint8_t>(), c->n,
                                                          cnt.as<unsigned long long>());
    GS_CUDA(c, cudaGetLastError());
    unsigned long long h[4];
    GS_CUDA(c, cudaMemcpyAsync(h, cnt.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    GS_CUDA(c, cudaStreamSynchronize(c->stream));
    cnt.release();
    const int64_t w = static_cast<int64_t>(h[1]), g = static_cast<int64_t>(h[2]);
    const int64_t tissue = w + g;
    if (tissue == 0) return fail(c, GS_EDATA, "matter_fractions: volume contains no tissue voxels");
    *white = static_cast<double>(w) / tissue;  // imaging.cpp:163
    *gray = static_cast<double>(g) / tissue;
    return GS_OK;
}

}  // extern "C"
