// gs_kernels.cuh -- kernel entry points and their parameter blocks.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "gliosim_b200.h"
#include "gs_device.cuh"

namespace gs {

enum SolveMode : int {
    kModeRun = 0,      // n exponential-Euler steps on the resident state (integrator.cpp:122-134)
    kModePhi1v = 1,    // phi1v(t, A, b) (expact.cpp:101-153)
    kModeExpmv = 2,    // expmv(t, A, b) (expact.cpp:63-99)
    kModeApply = 3,    // y = A x (sparse.cpp:43-76)
};

// Device vectors, by index (the TMA descriptors are indexed the same way).
enum Buf : int { kBufU = 0, kBufG = 1, kBufF0 = 2, kBufF1 = 3, kBufT0 = 4, kBufT1 = 5, kBufOut = 6, kNumBufs = 7 };

// TMA z-slab pipeline geometry: a CTA owns tiles of kTmaTX x kTmaTY columns and
// streams their z-planes through a kTmaStages-deep shared-memory ring.
//
// Default: 32 x 32 tiles, 512 threads (16 warps), each thread one column and two rows.  The
// two-term sweep's T1 halo ring is then 128 points -- exactly warps 0-3, one ring warp per
// SM sub-partition (measured against 64 x 16 tiles, whose 160-point ring needs five warps:
// +1.8% at C4, +0.7% at C3).  A/B builds: -DGS_TILE64 (64 x 16), -DGS_TILE8 (64 x 8 tiles,
// 256 threads, two CTAs per SM).
#if defined(GS_TILE8)
constexpr int kTmaTX = 64;
constexpr int kTmaTY = 8;
constexpr int kSolveThreads = 256;
constexpr int kMinBlocks = 2;        // __launch_bounds__ of the TMA kernels: 2 CTAs/SM, 128 regs
#elif defined(GS_TILE64)
constexpr int kTmaTX = 64;
constexpr int kTmaTY = 16;
constexpr int kSolveThreads = 512;   // 16 warps: warp w owns tile row w, two columns per lane
constexpr int kMinBlocks = 1;
#else
constexpr int kTmaTX = 32;
constexpr int kTmaTY = 32;
constexpr int kSolveThreads = 512;   // 16 warps: warp w owns rows w and w + 16 (single-term sweep)
constexpr int kMinBlocks = 1;
#endif
constexpr int kTmaStages = 6;

// The halo box starts two voxels left of the tile: TMA needs the innermost start coordinate
// times the element size to be a multiple of 16 bytes (measured: x0-1 faults on sm_100a).
constexpr int kXHalo = 2;                                              // x halo (left/right)
constexpr int kXCols = kTmaTX + 2 * kXHalo;                            // halo row: x0-2 .. x0+65
#ifdef GS_XPAD
// two more (unused) columns per row: a 70-double pitch spreads the column ring's rows over
// more shared-memory banks (row stride 140 words: 2-way instead of 4-way conflicts)
constexpr int kXPitch = kXCols + 2;
#else
constexpr int kXPitch = kXCols;                                        // doubles per halo row
#endif
constexpr int kXBytes = ((kTmaTY + 2) * kXPitch * 8 + 127) / 128 * 128;  // halo plane tile
constexpr int kOBytes = kTmaTX * kTmaTY * 8;                            // own plane tile (fp64)
constexpr int kLBytes = kTmaTX * kTmaTY;                                // own plane tile (labels)
constexpr int kSlotBytes = kXBytes + 2 * kOBytes + kLBytes;
constexpr int kRingBytes = kTmaStages * kSlotBytes + 128;              // + barriers

// Two-term fused sweep (temporal blocking): T_{j+1} is computed on the tile plus a one-voxel
// halo and kept in a 3-plane shared ring, T_{j+2} on the tile; the input therefore needs a
// two-voxel halo in x, y and z.
#ifdef GS_TILE8
constexpr int k2Stages = 7;
#elif defined(GS_STAGES8)
constexpr int k2Stages = 8;  // A/B: the eight-stage ring with rotating slot indices
#else
// six stages: the z-loop unrolled by six has compile-time slot indices (sweep2_tma); measured
// against eight stages with rotating indices: +1.0% at C4, +1.2% at C3, +2.6% at C5 -- two
// planes in flight beyond the four in use are enough lead at ~1 us per plane
constexpr int k2Stages = 6;
#endif
constexpr int k2XRows = kTmaTY + 4;                                     // y halo 2
constexpr int k2XBytes = (k2XRows * kXPitch * 8 + 127) / 128 * 128;    // 20 x 68 doubles
constexpr int k2BRows = kTmaTY + 2;                                     // y halo 1
constexpr int k2BBytes = (k2BRows * kXPitch * 8 + 127) / 128 * 128;    // 18 x 68 doubles
constexpr int kLHaloX = 16;                                             // u8 box: 16-byte aligned start
constexpr int kLPitch = kTmaTX + 2 * kLHaloX;                           // 96 labels per halo row
constexpr int k2LBytes = ((kTmaTY + 2) * kLPitch + 127) / 128 * 128;   // 18 x 96 labels
// F (own, next-kind) and b/gamma (halo, first-kind) are never needed by the same sweep: one region.
constexpr int k2FBBytes = kOBytes > k2BBytes ? kOBytes : k2BBytes;
constexpr int k2SlotBytes = k2XBytes + k2FBBytes + k2LBytes;
constexpr int kT1Pitch = kXPitch;  // same pitch as the X tile: T1, b/gamma and X offsets differ by constants
constexpr int kT1Rows = kTmaTY + 2;
constexpr int kT1Bytes = kT1Rows * kT1Pitch * 8;
constexpr int kT1Planes = 3;  // T1(z+1) is written while T1(z-1) is read; T1(z) is kept for the next iteration
constexpr int k2RingBytes = k2Stages * k2SlotBytes + kT1Planes * kT1Bytes + 128;
// implicit-X ring (a stage's first sweep reads f = F + T): F and T halo-2 tiles per slot
#ifdef GS_TILE8
constexpr int k2IStages = 4;
#elif defined(GS_XPAD)
constexpr int k2IStages = 5;
#else
constexpr int k2IStages = 6;
#endif
constexpr int k2ISlotBytes = 2 * k2XBytes + k2FBBytes + k2LBytes;
constexpr int k2IRingBytes = k2IStages * k2ISlotBytes + kT1Planes * kT1Bytes + 128;

// Three-term fused sweep: T_{j+1} on the tile plus a two-voxel ring (4-plane shared ring),
// T_{j+2} on the tile plus a one-voxel ring (3-plane shared ring), T_{j+3} on the tile; the
// input needs a three-voxel halo.  X slots (input + labels) and F/b slots are separate rings:
// F is consumed two planes behind X, b/gamma at X's pace, and never both in one sweep.
constexpr int k3XHaloX = 4;                                             // x0-4: 16-byte aligned start
constexpr int k3XPitch = kTmaTX + 2 * k3XHaloX;                         // 72
constexpr int k3XRows = kTmaTY + 6;                                     // y halo 3
constexpr int k3XBytes = (k3XRows * k3XPitch * 8 + 127) / 128 * 128;    // 22 x 72 doubles
constexpr int k3LRows = kTmaTY + 4;                                     // labels, y halo 2
constexpr int k3LBytes = (k3LRows * kLPitch + 127) / 128 * 128;         // 20 x 96 labels
constexpr int k3XSlotBytes = k3XBytes + k3LBytes;
#ifdef GS_TILE8
constexpr int k3XStages = 5;
#else
constexpr int k3XStages = 7;
#endif
constexpr int k3BRows = kTmaTY + 4;                                     // b/gamma, y halo 2
constexpr int k3BBytes = (k3BRows * k3XPitch * 8 + 127) / 128 * 128;    // 20 x 72 doubles
constexpr int k3FBBytes = kOBytes > k3BBytes ? kOBytes : k3BBytes;
#ifdef GS_TILE8
constexpr int k3FBStages = 2;
#else
constexpr int k3FBStages = 3;
#endif
constexpr int k3T1Pitch = kTmaTX + 4;
constexpr int k3T1Rows = kTmaTY + 4;
constexpr int k3T1Bytes = k3T1Rows * k3T1Pitch * 8;
constexpr int k3T1Planes = 4;
constexpr int k3T2Pitch = kTmaTX + 2;
constexpr int k3T2Rows = kTmaTY + 2;
constexpr int k3T2Bytes = k3T2Rows * k3T2Pitch * 8;
constexpr int k3T2Planes = 3;
constexpr int k3RingBytes = k3XStages * k3XSlotBytes + k3FBStages * k3FBBytes + k3T1Planes * k3T1Bytes +
                            k3T2Planes * k3T2Bytes + 128;
constexpr int kMaxRing0 = kRingBytes > k2RingBytes ? kRingBytes : k2RingBytes;
constexpr int kMaxRing = kMaxRing0 > k2IRingBytes ? kMaxRing0 : k2IRingBytes;
constexpr int kDynSmemBytes = kMaxRing > k3RingBytes ? kMaxRing : k3RingBytes;
// the Taylor kernel's block-reduction scratch (16 x 6 doubles) at the end of the dynamic
// region: past every TMA-written byte of every ring (the implicit ring's T1 planes, generic)
constexpr int kRedOffset = kDynSmemBytes - 128 - 768;  // (kSolveThreads / 32) x 6 doubles <= 768 B
static_assert(kRedOffset >= k2IStages * k2ISlotBytes && kRedOffset >= k2Stages * k2SlotBytes &&
                  kRedOffset >= kTmaStages * kSlotBytes && kRedOffset >= k3XStages * k3XSlotBytes + k3FBStages * k3FBBytes,
              "reduction scratch overlaps a TMA-written region");
static_assert(kDynSmemBytes + 2336 <= 232448, "dynamic + static shared memory over the 227 KB block limit");

constexpr int kXchgCtas = 160;   // CTAs of one (virtual) Taylor grid the maxima exchange can hold
constexpr int kXchgWords = 2 * kXchgCtas * kXchgCtas * 2;  // [set][inbox of CTA][from CTA][2 words]

// Device-resident control block shared by the kernels of one launch sequence.
struct Ctrl {
    double bnorm, gamma, prev0;
    int branch;           // 0 Taylor, 1 t == 0, 2 ||b||_1 == 0, 3 small norm
    int status, detail;   // gs_status of the first failure (later kernels return at once)
    int fres, tres;       // Taylor result: F[fres] (+ T[tres] when implicit)
    unsigned int ticket;  // last-block-done counter (metrics)
    int ntrace;
    int step;             // current step of a graph-replayed run (kernels launched with step < 0)
    // exact sequential sums (gs_seqsum.cuh): [0] ||b||_1, [1] the bordered column sum
    double seq[2];
    unsigned seq_ticket[2], seq_ticket2[2], seq_flags[2];
    unsigned border_ticket;
    int coln_need;        // the tree column sum does not settle (s, m): the exact one is required
    unsigned xround;      // rounds of the maxima exchange so far (xchg_keys4), across launches
    int last_terms;       // Taylor terms of the last step (ensemble: longest members first)
};

struct SolveParams {
    // TMA descriptors (64-byte aligned by type): halo-box and own-box maps per vector, labels
    CUtensorMap xmap[kNumBufs];
    CUtensorMap omap[kNumBufs];
    CUtensorMap x2map[kNumBufs];   // halo-2 boxes (fused two-term sweep)
    CUtensorMap x3map[kNumBufs];   // halo-3 boxes (fused three-term sweep)
    CUtensorMap b3map;             // b/gamma (buffer G) with a two-voxel halo
    CUtensorMap lmap;
    CUtensorMap l2map;             // labels with a one-voxel halo
    CUtensorMap l3map;             // labels with a two-voxel halo
    StencilOp op;
    int use_tma;
    int fuse;               // Taylor terms per fused TMA sweep: 2 or 3
    int mode;
    int n_steps;
    int want_metrics;
    int grid_blocks;
    int lock_groups;        // TMA sweeps: CTA groups marching z in lockstep (0 = even split; cta_work)
    int lock_zm;            // z-extent of the lockstep groups; the rest is split evenly
    int exact_max;          // two-term sweeps: 0 bounding maxima + exact fallback, 1 always exact, 2 always rerun
    double rho, tau, tol;   // tau doubles as t for phi1v / expmv
    double anorm;           // exact ||A||_1 (computed once by the norm kernel)
    double rtab[kMaxDegree + 1];  // r_m, m = 1..55, host libm (expact.cpp:47-48)
    double* buf[kNumBufs];
    // compute_metrics (integrator.cpp:65-89)
    double origin[3], center[3], h, front_threshold;
    double* metrics;        // [(n_steps+1)*4]
    gs_step_info* infos;    // [n_steps] or nullptr
    // cross-CTA scratch
    double* part_b;         // [grid] block partial sums of |b|
    double* part_c;         // [grid] block partial sums of |b/gamma|
    double* part_u;         // [grid] block partial sums of u (metrics)
    // exact sequential sums (gs_seqsum.cuh): per-tile approximate sums / prefixes, per-CTA
    // item lists (seq::Item[kSeqItemCap] each) and their {count, overflow} words
    double* seq_tsum;
    void* seq_items;
    int* seq_counts;
    int seq_tiles;
    int seq_exact;          // 1: the two sums are the reference's sequential ones; 0: tree sums (A/B)
    unsigned long long* slots;   // [3][8] rotating max slots for per-term reductions (+ the 2-D kernel's: kSlotWords)
    unsigned long long* mslots;  // [2][4] metric max/min/r2 slots (step parity)
    // Bounded two-term sweeps: the per-sweep maxima exchange that is also the sweep's grid
    // barrier (xchg_keys4; kXchgWords words cleared per run; nullptr: atomicMax slots + grid barrier)
    unsigned long long* xchg;
    // 2-D grids with one resident CTA per tile (gs_flat2d.cuh): 2 (k2dK + 1) N-vectors of scratch
    int use_2d;
    double* x2d;
    Ctrl* ctrl;
    unsigned long long* trace;  // optional phase trace: (tag, globaltimer ns) pairs
    int trace_cap;
};

// phase tags of the optional trace (leader's view, recorded after each grid barrier)
enum TraceTag : int { kTrMetrics0 = 1, kTrRhs = 2, kTrBorder = 3, kTrFusedFirst = 4, kTrFusedNext = 5, kTrFixup = 6,
                      kTrUpdate = 7, kTrTerm = 8, kTrBranch = 9, kTrBorderIn = 10, kTrTaylorIn = 11,
                      kTrUpdateIn = 12, kTrPrepIn = 13, kTrStart = 15 };

// K1: resample + classify (imaging.cpp:65-72, 118-141)
__global__ void material_kernel(const uint8_t* stack, int w, int hgt, int slices, int nx, int ny, int nz,
                                int t_air, int t_white, int t_gray, uint8_t* labels);
// K3: exact 1-norm of the stencil operator (sparse.cpp:36-40), result as ordered bits
__global__ void colsum_norm_kernel(StencilOp op, unsigned long long* out_bits);
// Exact 1-norm of a generic operator from its transpose (CSC, rows ascending within a column):
// one thread per column sums |a| in the CSR storage order the reference's constructor walks.
__global__ void csc_norm_kernel(int64_t n, const int64_t* csc_offs, const double* csc_absvals,
                                unsigned long long* out_bits);
// Per-voxel D(x) reconstruction (for gs_get_diffusion in palette mode)
__global__ void expand_palette_kernel(const uint8_t* pal, const double* dtab, int64_t n, double* d);
__global__ void label_count_kernel(const uint8_t* labels, int64_t n, unsigned long long* counts);
// The exponential-Euler step as a launch sequence (gs_solve.cu):
//   [metrics_kernel] -> per step: prep_kernel -> border_kernel -> taylor_kernel (cooperative) -> update_kernel
__global__ void metrics_kernel(const __grid_constant__ SolveParams p);
__global__ void prep_kernel(const __grid_constant__ SolveParams p, int step);
__global__ void border_kernel(const __grid_constant__ SolveParams p, int prep_blocks, int step);
// The reference's sequential sums (gs_seqsum.cuh), which = 0 ||b||_1, 1 the bordered column sum:
// tile pass, then item pass + composer (last CTA); result in ctrl->seq[which].
__global__ void seqsum_tiles_kernel(const __grid_constant__ SolveParams p, int which);
__global__ void seqsum_items_kernel(const __grid_constant__ SolveParams p, int which);
constexpr int kSeqTileElems = kSolveThreads * 8;  // elements per tile (kSeqTile in gs_solve.cu)
constexpr int kSeqItemBytes = 40;                 // sizeof(seq::Item)
constexpr int kSeqItemsPerCta = 512;              // kSeqItemCap
constexpr int kSeqMaxCtas = 1024;                 // kSeqMaxLists: the composer's list index
// Small grids: whole runs in one thread-block cluster (gs_cluster.cu).
constexpr int kClusterCTAs = 16;  // non-portable cluster size (opt-in attribute)
struct ClusterParams {
    StencilOp op;            // palette mode: pal + wtab
    int n_steps, want_metrics;
    int seq_exact;           // 1: the reference's sequential sums (gs_seqsum.cuh); 0: rank-order tree sums
    int64_t slice, halo;     // voxels per CTA, halo width (one plane, or one row in 2-D)
    double rho, tau, tol, anorm;
    double rtab[kMaxDegree + 1];
    double* u;               // resident state: read at the start, written at the end
    double* metrics;         // [(n_steps+1)*4] or nullptr
    gs_step_info* infos;     // [n_steps] or nullptr
    Ctrl* ctrl;
    double origin[3], center[3], h, front_threshold;
};
// The exact sums' gathered item lists (gs_cluster.cu) alias the four Taylor vectors F0..T1,
// idle while ||b||_1 and the column sum are formed: 16 ranks x 32 items + 8 padding, 56 bytes
// each (kind, B, d0, d1, lo, hi, start/len).
constexpr int kClItemCap = 32;
constexpr int kClAll = kClusterCTAs * kClItemCap + 8;
constexpr int64_t kClGatherDoubles = (static_cast<int64_t>(kClAll) * 56 + 7) / 8;
// Offset (doubles) of b/gamma: U, then F0, F1, T0, T1 -- padded to hold the gather.
__host__ __device__ inline int64_t cluster_b_offset(int64_t slice, int64_t halo) {
    const int64_t hs = slice + 2 * halo;
    // (+2: the gather starts at the first 16-byte boundary of F0, which may be 8 bytes in)
    return hs + (4 * hs > kClGatherDoubles + 2 ? 4 * hs : kClGatherDoubles + 2);
}
// Dynamic shared memory of cluster_run_kernel per CTA (5 haloed vectors, b/gamma, labels,
// neighbour masks).
inline size_t cluster_smem_bytes(int64_t slice, int64_t halo) {
    return static_cast<size_t>(cluster_b_offset(slice, halo) + slice) * 8 +
           2 * ((static_cast<size_t>(slice) + 15) / 16) * 16;
}
__global__ void cluster_run_kernel(const __grid_constant__ ClusterParams p);

// ctrl->step += 1: closes one step of a CUDA-graph replayed run.
__global__ void advance_kernel(Ctrl* ctrl);
// Taylor kernel as a launchable handle: FUSE = 2 or 3 Taylor terms per TMA pass, 4 = two
// terms with the past-the-grid planes skipped (thin grids).
const void* taylor_kernel_fn(int fuse);
// The resident-tile Taylor kernel of 2-D grids (gs_flat2d.cuh): cooperative, one CTA per
// 32 x 32 tile, k2dSmemBytes of dynamic shared memory; nullptr in builds without 512 threads.
#ifndef GS_2D_K
#define GS_2D_K 4
#endif
constexpr int k2dK = GS_2D_K;  // Taylor terms per round (one grid barrier): 2..6
// max slots: [3][8] of the sweeps, then [3][kSlots2d] of the 2-D kernel's rounds (2K maxima each)
constexpr int kSlots2dBase = 24, kSlots2d = 16, kSlotWords = kSlots2dBase + 3 * kSlots2d;
constexpr int k2dSmemBytes = (k2dK + 3) * (32 + 2 * k2dK) * (32 + 2 * k2dK) * 8;
const void* taylor2d_kernel_fn();
__global__ void update_kernel(const __grid_constant__ SolveParams p, int step);

// Ensemble (C5) forms of the step's kernels: one launch serves every member; P is a device
// array of the members' SolveParams (TMA descriptors read from global memory).  CTA b of the
// streaming/prep launches works for member b / cpm as CTA b % cpm of cpm.  The Taylor kernel
// is cooperative: gridDim.x / group CTA groups take members from a queue, each running one
// member's Taylor loop on its group with a software group barrier.  ctl: 4 words per group
// plus the queue head, zeroed before each launch, then n_members words of the queue's order
// (ens_order_kernel: members by their last step's Taylor terms, most first).
__global__ void ens_metrics_kernel(const SolveParams* P, int cpm);
__global__ void ens_prep_kernel(const SolveParams* P, int cpm, int step);
__global__ void ens_border_kernel(const SolveParams* P, int cpm, int prep_blocks, int step);
__global__ void ens_update_kernel(const SolveParams* P, int cpm, int step);
__global__ void ens_seqsum_tiles_kernel(const SolveParams* P, int cpm, int which);
__global__ void ens_seqsum_items_kernel(const SolveParams* P, int cpm, int which);
__global__ void ens_order_kernel(const SolveParams* P, int n_members, unsigned* order);
const void* ens_taylor_kernel_fn(int fuse);  // fuse 2 or 4 (args: P, n_members, group, border_blocks, step, ctl, order, extra)
inline int ens_ctl_words(int groups) { return 4 * groups + 1; }

}  // namespace gs
