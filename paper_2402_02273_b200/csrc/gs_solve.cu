// gs_solve.cu -- the persistent exponential-Euler kernel (sm_100a).
//
// One cooperative launch runs whole exponential-Euler steps (integrator.cpp:52-63) for
// every step of a run (integrator.cpp:122-134):
//
//   K2  RHS sweep        g = A u + rho u (1-u), ||g||_1                (integrator.cpp:54-57)
//   --  bordered column  g <- g/gamma, sum|g/gamma|; (s, m) on device   (expact.cpp:110-142, 29-61)
//   K4  Taylor terms     T_j = (t/s)/j * (A~ T_{j-1}); f += T_j; ||T||, ||f||; stop test
//                        (expact.cpp:79-97) -- one HBM pass per term
//   K5  update + metrics u <- u + tau*(gamma/tau)*f; compute_metrics   (integrator.cpp:58-61, 65-89)
//
// Phases are separated by grid-wide barriers (cooperative groups); every CTA evaluates the
// same scalar control flow from the same reduced values, so the (s, m) choice and the
// early-termination decisions are taken identically everywhere with no host round trip.
//
// Stencil sweeps stream z-planes of a kTmaTX x kTmaTY column tile through a
// kTmaStages-deep shared-memory ring filled by TMA (cp.async.bulk.tensor, halo tiles with
// out-of-bounds zero fill = the missing Neumann neighbours); each thread keeps the z-1/z/z+1
// values of its columns in registers and takes its in-plane neighbours from shared memory.
// Each CTA owns a fixed, balanced, contiguous range of tile-planes (one CTA per SM).
// Shapes the TMA path cannot describe (nx % 16 != 0, fp64-D mode) use an L1-cached
// fallback sweep with identical arithmetic.
#include <cooperative_groups.h>

#include <cstdio>
#include <type_traits>

#include "gs_kernels.cuh"
#include "gs_tma.cuh"

namespace cg = cooperative_groups;

namespace gs {

namespace {

// Virtual grid: this CTA's index and the CTA count of the work it belongs to.  A plain launch
// is its own virtual grid; the ensemble kernels cut one launch into per-member virtual grids
// (a CTA group per member, ens_* below).  Set first thing by every kernel (vgrid_set).
__shared__ int s_vgrid[2];
__device__ __forceinline__ void vgrid_set(int cta, int ncta) {
    if (threadIdx.x == 0) {
        s_vgrid[0] = cta;
        s_vgrid[1] = ncta;
    }
    __syncthreads();
}
__device__ __forceinline__ int vcta() { return s_vgrid[0]; }
__device__ __forceinline__ int vncta() { return s_vgrid[1]; }

struct SmemCore {
    double wtab[256];
    double bcast[4];
    uint64_t bar1[kTmaStages];   // single-term ring
    uint64_t bar2[k2Stages];     // fused two-term rings (the implicit-X ring uses the first k2IStages)
    uint64_t bar3x[k3XStages];   // fused three-term ring: input + labels
    uint64_t bar3f[k3FBStages];  // fused three-term ring: F or b/gamma
};

// Static shared memory of the streaming kernels.
struct Smem : SmemCore {
    double red[kSolveThreads / 32][6];
};

// The Taylor kernel's: its reduction scratch lives in dynamic shared memory (kRedOffset,
// only ever touched by generic stores and idle during sweeps), which leaves the largest
// TMA ring (k2IRingBytes) room under the 227 KB per-block limit.
struct SmemT : SmemCore {
    double (*red)[6];
};

struct Ring {
    unsigned char* base;
    uint64_t* bar;
    __device__ double* x(int s) const { return reinterpret_cast<double*>(base + s * kSlotBytes); }
    __device__ double* f(int s) const { return reinterpret_cast<double*>(base + s * kSlotBytes + kXBytes); }
    __device__ double* b(int s) const { return reinterpret_cast<double*>(base + s * kSlotBytes + kXBytes + kOBytes); }
    __device__ uint8_t* l(int s) const { return base + s * kSlotBytes + kXBytes + 2 * kOBytes; }
};

// Block reduction of up to 4 values with a fixed shape; result valid in thread 0.
template <int K, bool kMax, class S>
__device__ __forceinline__ void block_reduce(double (&v)[K], S& sm) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = kMax ? warp_max(v[q]) : warp_sum(v[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < K; ++q) sm.red[wid][q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            double a = sm.red[0][q];
            for (int w = 1; w < kSolveThreads / 32; ++w)
                a = kMax ? nan_dropping_max(a, sm.red[w][q]) : __dadd_rn(a, sm.red[w][q]);
            v[q] = a;
        }
    }
    __syncthreads();
}

// Maxima exchange of the bounded two-term sweeps: the sweep's grid barrier and the all-reduce
// (max) of its four bounding maxima in ONE round trip through L2, in place of atomicMax slots
// + grid barrier + slot reads (three).
//   push   thread e < G of CTA c stores c's block maxima into CTA e's inbox, entry c;
//   poll   the same thread waits for entry e of its own CTA's inbox (lines only this CTA
//          reads: no hot spot), then a block max over the entries gives every thread the grid
//          maxima.
// Seeing CTA e's entry means CTA e has finished its sweep (each pusher fences after the block
// barrier that follows the sweep, then stores; the poller fences after its loads), so this is
// the barrier between sweeps as well.  A bounding maximum travels as its key, the high word of
// a non-negative double with a zero low word (key_lower): 31 bits, two per 64-bit word, whose
// two spare bits carry the round's tag.  The two entry sets alternate by round; tags cycle
// 1, 2, 3 over the uses of a set and 0 is the cleared state (setup_solve), so an entry of the
// set's previous use never passes for the current one -- a CTA cannot push round r + 2 before
// every CTA has polled round r, since it first has to see every CTA's round r + 1 entry.  The
// round counter lives in the control block across launches (ctrl->xround).
template <class S>
__device__ __forceinline__ void xchg_keys4(const SolveParams& p, S& sm, double (&mx)[5], unsigned xr) {
    const int G = vncta(), me = vcta();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long* set = p.xchg + static_cast<size_t>(xr & 1u) * (kXchgCtas * kXchgCtas * 2);
    const unsigned tag = 1u + ((xr >> 1) % 3u);
    const unsigned t_hi = (tag >> 1) << 31, t_lo = (tag & 1u) << 31;
    unsigned* s1 = reinterpret_cast<unsigned*>(&sm.red[0][0]);  // [warps][4] block stage
    unsigned* s2 = s1 + (kSolveThreads / 32) * 4;               // [<= 5][4] grid stage
    unsigned k[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) k[q] = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(__double2hiint(mx[q])));
    if (lane == 0) *reinterpret_cast<uint4*>(s1 + 4 * wid) = make_uint4(k[0], k[1], k[2], k[3]);
    __syncthreads();  // also: every thread's sweep writes precede the pushers' fences
    k[0] = k[1] = k[2] = k[3] = 0u;
    if (tid < G) {
#pragma unroll
        for (int w = 0; w < kSolveThreads / 32; ++w) {
            const uint4 v = *reinterpret_cast<const uint4*>(s1 + 4 * w);
            k[0] = max(k[0], v.x);
            k[1] = max(k[1], v.y);
            k[2] = max(k[2], v.z);
            k[3] = max(k[3], v.w);
        }
        const unsigned long long w0 = (static_cast<unsigned long long>(k[0] | t_hi) << 32) | (k[1] | t_lo);
        const unsigned long long w1 = (static_cast<unsigned long long>(k[2] | t_hi) << 32) | (k[3] | t_lo);
        __threadfence();
        volatile unsigned long long* out = set + (static_cast<size_t>(tid) * kXchgCtas + me) * 2;
        out[0] = w0;
        out[1] = w1;
        const volatile unsigned long long* in = set + (static_cast<size_t>(me) * kXchgCtas + tid) * 2;
        const unsigned long long tmask = (1ull << 63) | (1ull << 31);
        const unsigned long long twant = (static_cast<unsigned long long>(t_hi) << 32) | t_lo;
        unsigned long long a, b;
        do {
            a = in[0];
            b = in[1];
        } while ((a & tmask) != twant || (b & tmask) != twant);
        __threadfence();
        k[0] = static_cast<unsigned>(a >> 32) & 0x7fffffffu;
        k[1] = static_cast<unsigned>(a) & 0x7fffffffu;
        k[2] = static_cast<unsigned>(b >> 32) & 0x7fffffffu;
        k[3] = static_cast<unsigned>(b) & 0x7fffffffu;
    }
    const int nw = (G + 31) >> 5;
    if (wid < nw) {
#pragma unroll
        for (int q = 0; q < 4; ++q) k[q] = __reduce_max_sync(0xffffffffu, k[q]);
        if (lane == 0) *reinterpret_cast<uint4*>(s2 + 4 * wid) = make_uint4(k[0], k[1], k[2], k[3]);
    }
    __syncthreads();
    k[0] = k[1] = k[2] = k[3] = 0u;
    for (int w = 0; w < nw; ++w) {
        const uint4 v = *reinterpret_cast<const uint4*>(s2 + 4 * w);
        k[0] = max(k[0], v.x);
        k[1] = max(k[1], v.y);
        k[2] = max(k[2], v.z);
        k[3] = max(k[3], v.w);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) mx[q] = __hiloint2double(static_cast<int>(k[q]), 0);
    mx[4] = 0.0;
    __syncthreads();  // the scratch is free again
}

// Deterministic sum of the per-CTA partials; every CTA computes the same value.
template <class S>
__device__ double grid_sum(const double* part, int nb, S& sm) {
    if (threadIdx.x < 32) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < nb; b += 32) acc = __dadd_rn(acc, __ldcg(part + b));
        acc = warp_sum(acc);
        if (threadIdx.x == 0) sm.bcast[0] = acc;
    }
    __syncthreads();
    const double r = sm.bcast[0];
    __syncthreads();
    return r;
}

#include "gs_seqsum.cuh"

// ------------------------------------------------------------------------------------------
// Exact sequential sums (gs_seqsum.cuh): which = 0 ||b||_1 of G (before the border pass),
// which = 1 the bordered column sum of G = b/gamma (after it).
// ------------------------------------------------------------------------------------------

constexpr int kSeqMaxLists = 1024;  // CTA lists the composer can index (virtual grids <= 2 x SMs)
static_assert(kSeqTile == kSeqTileElems && sizeof(seq::Item) == kSeqItemBytes && kSeqItemCap == kSeqItemsPerCta &&
                  kSeqMaxLists == kSeqMaxCtas,
              "gs_kernels.cuh mirrors the seqsum layout");

__device__ __forceinline__ bool seq_skip(const SolveParams& p, int which) {
    if (__ldcg(&p.ctrl->status)) return true;
    if (which == 0) return false;
    // the column sum: only on the Taylor branch, and only when (s, m) or the step log needs it
    return __ldcg(&p.ctrl->branch) != 0 || (!p.infos && !__ldcg(&p.ctrl->coln_need));
}

// Pass 1: approximate per-tile sums (any order) and non-finite flags; the last CTA turns the
// tile sums into approximate exclusive prefixes (in place).
__device__ __forceinline__ void seqsum_tiles_body(const SolveParams& p, int which) {
    __shared__ SeqSmem sm;
    __shared__ double s_part[16][kSolveThreads / 32];
    if (seq_skip(p, which)) return;
    Ctrl* ctrl = p.ctrl;
    const double* X = p.buf[kBufG];
    const int64_t n = p.op.n;
    const int tiles = p.seq_tiles;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned flags = 0;
    // tiles vcta(), vcta() + vncta(), ...: warp partials in shared memory, 16 tiles per barrier;
    // the loads of four tiles are issued before any of their reductions
    constexpr int kG = 2;
    for (int t0 = vcta(); t0 < tiles; t0 += 16 * vncta()) {
        for (int k0 = 0; k0 < 16; k0 += kG) {
            double v[kG][kSeqEPT];
#pragma unroll
            for (int g = 0; g < kG; ++g) {
                const int t = t0 + (k0 + g) * vncta();
                const int64_t base = static_cast<int64_t>(t) * kSeqTile + threadIdx.x;
                if (t < tiles && static_cast<int64_t>(t + 1) * kSeqTile <= n) {  // whole tile: no predicates
#pragma unroll
                    for (int j = 0; j < kSeqEPT; ++j) v[g][j] = X[base + static_cast<int64_t>(j) * kSolveThreads];
                } else {
#pragma unroll
                    for (int j = 0; j < kSeqEPT; ++j) {
                        const int64_t i = base + static_cast<int64_t>(j) * kSolveThreads;
                        v[g][j] = t < tiles && i < n ? X[i] : 0.0;
                    }
                }
            }
            double s[kG];
#pragma unroll
            for (int g = 0; g < kG; ++g) {
                s[g] = 0.0;
#pragma unroll
                for (int j = 0; j < kSeqEPT; ++j) {
                    const double x = fabs(v[g][j]);
                    flags |= isnan(x) ? seq::kHasNaN : (isinf(x) ? seq::kHasInf : 0u);
                    s[g] = __dadd_rn(s[g], x);
                }
            }
#pragma unroll
            for (int g = 0; g < kG; ++g) {
                const double v = warp_sum(s[g]);
                if (lane == 0) s_part[k0 + g][w] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x < 16) {
            const int t = t0 + threadIdx.x * vncta();
            if (t < tiles) {
                double tot = 0.0;
                for (int q = 0; q < kSolveThreads / 32; ++q) tot = __dadd_rn(tot, s_part[threadIdx.x][q]);
                p.seq_tsum[t] = tot;
            }
        }
        __syncthreads();
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(&ctrl->seq_flags[which], flags);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        sm.last = atomicAdd(&ctrl->seq_ticket[which], 1u) == static_cast<unsigned>(vncta()) - 1;
    }
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    // approximate exclusive prefixes into seq_tsum[tiles ..]: thread i takes ceil(tiles/threads)
    // consecutive tiles, one block scan
    double* pre = p.seq_tsum + tiles;
    const int per = (tiles + kSolveThreads - 1) / kSolveThreads;
    const int lo = min(tiles, static_cast<int>(threadIdx.x) * per), hi = min(tiles, lo + per);
    double mine = 0.0;
    for (int t = lo; t < hi; ++t) mine = __dadd_rn(mine, __ldcg(p.seq_tsum + t));
    double run = seq_block_excl_sum(mine, sm, nullptr);
    for (int t = lo; t < hi; ++t) {
        pre[t] = run;
        run = __dadd_rn(run, __ldcg(p.seq_tsum + t));
    }
    if (threadIdx.x == 0) ctrl->seq_ticket[which] = 0u;
}

// s <- fl(s + |X[i]|) for i in [lo, hi): the reference's loop itself (fallback of the walk)
__device__ __noinline__ double seq_walk(double s, const double* X, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) s = __dadd_rn(s, fabs(__ldcg(X + i)));
    return s;
}

// Pass 2: per CTA, a contiguous range of tiles -> its list of run / raw items; the last CTA
// composes all lists in order into the exact sequential sum.
__device__ __forceinline__ void seqsum_items_body(const SolveParams& p, int which) {
    __shared__ SeqSmem sm;
    __shared__ int s_kind[kSolveThreads], s_B[kSolveThreads];
    __shared__ uint64_t s_d0[kSolveThreads], s_d1[kSolveThreads], s_lo[kSolveThreads], s_hi[kSolveThreads];
    __shared__ longlong2 s_pos[kSolveThreads];
    __shared__ int s_pref[kSeqMaxLists + 1];
    if (seq_skip(p, which)) return;
    Ctrl* ctrl = p.ctrl;
    const double* X = p.buf[kBufG];
    const int64_t n = p.op.n;
    const int tiles = p.seq_tiles;
    const int nc = vncta(), c = vcta();
    const int tpc = (tiles + nc - 1) / nc;
    const int t_lo = min(tiles, c * tpc), t_hi = min(tiles, t_lo + tpc);
    seq::Item* items = static_cast<seq::Item*>(p.seq_items) + static_cast<size_t>(c) * kSeqItemCap;
    const unsigned fl = __ldcg(&ctrl->seq_flags[which]);
    if (threadIdx.x == 0) seq_open_reset(sm);
    __syncthreads();
    // tile t's data (thread-contiguous kSeqEPT elements) and its prefix / sum are loaded one
    // tile ahead
    double xn[kSeqEPT], pn = 0.0, sn = 0.0;
    const double* pre = p.seq_tsum + tiles;
    auto load_tile = [&](int t) {
        const int64_t b = static_cast<int64_t>(t) * kSeqTile + static_cast<int64_t>(threadIdx.x) * kSeqEPT;
        if (b + kSeqEPT <= n) {
            const double2* X2 = reinterpret_cast<const double2*>(X + b);
#pragma unroll
            for (int j = 0; j < kSeqEPT / 2; ++j) {
                const double2 v = X2[j];
                xn[2 * j] = v.x;
                xn[2 * j + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kSeqEPT; ++j) xn[j] = b + j < n ? X[b + j] : 0.0;
        }
        pn = __ldcg(pre + t);
        sn = __ldcg(p.seq_tsum + t);
    };
    if (fl == 0 && t_lo < t_hi) load_tile(t_lo);
    for (int t = t_lo; t < t_hi && fl == 0; ++t) {
        const int64_t base = static_cast<int64_t>(t) * kSeqTile;
        const int cnt = static_cast<int>(min(static_cast<int64_t>(kSeqTile), n - base));
        double x[kSeqEPT];
#pragma unroll
        for (int j = 0; j < kSeqEPT; ++j) x[j] = xn[j];
        const double a_tile = pn, t_sum = sn;
        if (t + 1 < t_hi) load_tile(t + 1);
        // the whole tile in one binade (pass 1's tile sum, widened by delta): one run
        const int bt = seq::binade(__dmul_rn(a_tile, 1.0 - seq::kDelta));
        const double a_end = __dmul_rn(__dadd_rn(a_tile, t_sum), 1.0 + seq::kDelta);
        if (isfinite(a_end) && bt == seq::binade(a_end)) {
#pragma unroll
            for (int j = 0; j < kSeqEPT; ++j) x[j] = fabs(x[j]);
            seq_fast_tile<kSeqEPT>(sm, x, bt, base, items, kSeqItemCap, t & 1);
        } else {
            __syncthreads();  // thread 0's merge of a previous fast tile is visible
            seq_tile_items<kSeqEPT>(sm, x, base, cnt, a_tile, items, kSeqItemCap);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int k = sm.items;
        if (fl == 0 && t_lo < t_hi) k = seq_close(sm, min(n, static_cast<int64_t>(t_hi) * kSeqTile), items, kSeqItemCap);
        p.seq_counts[2 * c] = min(k, kSeqItemCap);
        p.seq_counts[2 * c + 1] = k > kSeqItemCap;
        __threadfence();
        sm.last = atomicAdd(&ctrl->seq_ticket2[which], 1u) == static_cast<unsigned>(nc) - 1;
    }
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    // ---- composer (last CTA): walk the lists in order from s = 0
    long long t_c0 = clock64(), t_walk = 0;
    double s = 0.0;
    if (fl & seq::kHasNaN) {
        s = __longlong_as_double(0x7ff8000000000000ll);
    } else if (fl & seq::kHasInf) {
        s = __longlong_as_double(0x7ff0000000000000ll);
    } else {
        // items per list (an overflowed list counts as one pseudo-item: its whole range)
        int tot = 0;
        for (int c0 = 0; c0 < nc; c0 += kSolveThreads) {
            const int cc = c0 + threadIdx.x;
            int cnt = 0;
            if (cc < nc) cnt = __ldcg(p.seq_counts + 2 * cc + 1) ? 1 : __ldcg(p.seq_counts + 2 * cc);
            int t2;
            const int ex = seq_block_excl_int(cnt, sm, &t2);
            if (cc < nc && cc < kSeqMaxLists) s_pref[cc] = tot + ex;
            tot += t2;
        }
        if (threadIdx.x == 0) {
            s_pref[min(nc, kSeqMaxLists)] = tot;
            sm.st = SeqState{-1022, 0ull};  // s = +0
            sm.fin = true;
        }
        __syncthreads();
        const seq::Item* all = static_cast<const seq::Item*>(p.seq_items);
        for (int g0 = 0; g0 < tot; g0 += kSolveThreads) {
            const int g = g0 + threadIdx.x;
            int kd = seq::kEmpty, bq = 0;
            uint64_t q0 = 0ull, q1 = 0ull;
            longlong2 qp = make_longlong2(0, 0);
            if (g < tot) {
                int lo = 0, hi = min(nc, kSeqMaxLists) - 1;  // list of item g: last pref <= g
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_pref[mid] <= g) lo = mid;
                    else hi = mid - 1;
                }
                if (__ldcg(p.seq_counts + 2 * lo + 1)) {
                    const int64_t b0 = static_cast<int64_t>(lo) * tpc * kSeqTile;
                    const int64_t e0 = min(n, static_cast<int64_t>(min(tiles, (lo + 1) * tpc)) * kSeqTile);
                    kd = seq::kMixed;
                    qp = make_longlong2(b0, e0 - b0);
                } else {
                    const seq::Item* it = all + static_cast<size_t>(lo) * kSeqItemCap + (g - s_pref[lo]);
                    kd = __ldcg(&it->kind);
                    bq = __ldcg(&it->B);
                    q0 = __ldcg(&it->d0);
                    q1 = __ldcg(&it->d1);
                    qp = make_longlong2(__ldcg(&it->start), __ldcg(&it->len));
                }
            }
            {
                s_kind[threadIdx.x] = kd;
                s_B[threadIdx.x] = bq;
                seq_stage(kd, bq, q0, q1, s_d0[threadIdx.x], s_d1[threadIdx.x], s_lo[threadIdx.x], s_hi[threadIdx.x]);
                s_pos[threadIdx.x] = qp;
            }
            __syncthreads();
            if (threadIdx.x == 0 && sm.fin) {
                const long long tw = clock64();
                uint64_t bits = static_cast<uint64_t>(__double_as_longlong(sm.st.value()));
                sm.fin = seq_walk_batch(bits, s_kind, s_B, s_d0, s_d1, s_lo, s_hi, s_pos, min(kSolveThreads, tot - g0),
                                        [&](double a, int64_t lo, int64_t hi) { return seq_walk(a, X, lo, hi); },
                                        p.seq_exact > 1);
                sm.st.set(__longlong_as_double(static_cast<long long>(bits)));
                t_walk += clock64() - tw;
            }
            __syncthreads();
        }
        s = sm.fin ? sm.st.value() : __longlong_as_double(0x7ff0000000000000ll);
        if (p.seq_exact > 1 && threadIdx.x == 0)
            printf("seqsum %d: %d lists, %d items, sum %a; composer %lld cycles, walk %lld\n", which, nc, tot, s,
                   clock64() - t_c0, t_walk);
    }
    if (threadIdx.x == 0) {
        ctrl->seq[which] = s;
        ctrl->seq_flags[which] = 0u;
        ctrl->seq_ticket2[which] = 0u;
        __threadfence();
    }
}

__device__ __forceinline__ double slot_read(const unsigned long long* s) {
    return __longlong_as_double(static_cast<long long>(__ldcg(s)));
}

// select_params (expact.cpp:29-61) with the libm part (r_m) precomputed on the host;
// what remains is IEEE division, ceil, max, multiply and compare: bit-identical.
__device__ int select_params_dev(double norm_tA, const double* rtab, int* s_out, int* m_out) {
    if (!isfinite(norm_tA) || norm_tA < 0.0) return GS_EINVAL;
    *s_out = 1;
    *m_out = 1;
    if (norm_tA == 0.0) return GS_OK;
    double best_cost = -1.0;
    for (int m = 1; m <= kMaxDegree; ++m) {
        const double c = ceil(__ddiv_rn(norm_tA, rtab[m]));
        const double stages = (1.0 < c) ? c : 1.0;
        if (stages > 2e9) continue;
        const double cost = __dmul_rn(stages, static_cast<double>(m));
        if (best_cost < 0.0 || cost < best_cost) {
            best_cost = cost;
            *s_out = static_cast<int>(stages);
            *m_out = m;
        }
    }
    return best_cost < 0.0 ? GS_ENUMERIC : GS_OK;
}

// ------------------------------------------------------------------------------------------
// Sweeps
// ------------------------------------------------------------------------------------------

// Pointwise sweep: grid-stride over voxels, no neighbours.
template <class Body>
__device__ __forceinline__ void sweep_points(const StencilOp& op, Body&& body) {
    const int64_t stride = static_cast<int64_t>(vncta()) * blockDim.x;
    for (int64_t v = static_cast<int64_t>(vcta()) * blockDim.x + threadIdx.x; v < op.n; v += stride) body(v);
}

// Fallback stencil sweep (L1-cached loads, z-march in registers); used where TMA cannot
// describe the arrays.  Tiles of 32 x (blockDim/32) columns times z-chunks of op.zc planes.
template <class Body>
__device__ __forceinline__ void sweep_l1(const StencilOp& op, const double* X, const double* F, const double* B,
                                         const double* s_wtab, Body&& body) {
    const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
    const int ty_n = blockDim.x >> 5;
    const int64_t tiles = static_cast<int64_t>(op.tiles_x) * op.tiles_y;
    const int64_t vc = vcta(), vn = vncta();
    for (int64_t item = vc; item < op.n_items; item += vn) {
        const int64_t tile = item % tiles;
        const int chunk = static_cast<int>(item / tiles);
        const int i = static_cast<int>(tile % op.tiles_x) * 32 + lx;
        const int j = static_cast<int>(tile / op.tiles_x) * ty_n + ly;
        const bool act = i < op.nx && j < op.ny;
        const int z0 = chunk * op.zc;
        const int z1 = min(op.nz, z0 + op.zc);
        const int64_t colv = i + static_cast<int64_t>(j) * op.sy;
        double xm = 0.0, xc = 0.0;
        if (act) {
            xm = z0 > 0 ? X[colv + (z0 - 1) * op.sz] : 0.0;
            xc = X[colv + z0 * op.sz];
        }
        const bool hx0 = i > 0, hx1 = i < op.nx - 1, hy0 = j > 0, hy1 = j < op.ny - 1;
        for (int k = z0; k < z1; ++k) {
            const int64_t v = colv + k * op.sz;
            const bool hz0 = k > 0, hz1 = k < op.nz - 1;
            double xp = 0.0;
            if (act) {
                xp = hz1 ? X[v + op.sz] : 0.0;
                const double xxm = hx0 ? X[v - 1] : 0.0;
                const double xxp = hx1 ? X[v + 1] : 0.0;
                const double xym = hy0 ? X[v - op.sy] : 0.0;
                const double xyp = hy1 ? X[v + op.sy] : 0.0;
                const RowCoef rc = row_coef(op, s_wtab, v);
                const int cnt = hx0 + hx1 + hy0 + hy1 + hz0 + hz1;
                const double acc = row_apply(rc, cnt, xm, xym, xxm, xc, xxp, xyp, xp);
                body(v, acc, xc, F ? F[v] : 0.0, B ? B[v] : 0.0);
            }
            xm = xc;
            xc = xp;
        }
    }
}

// Work of this CTA in a TMA sweep: tile-planes q in [qb, qe) of a z-range [zb, zb + len),
// numbered q = tile * len + (z - zb), so a CTA marches z within a tile column.
//
// Default: the whole grid as one range, split evenly.  Lockstep (p.lock_groups = k > 0, set
// by the host when the grid holds k full planes of tiles, SolveParams): the first k*P CTAs
// form k groups of one CTA per tile; group j marches z-chunk j of [0, lock_zm), so every
// tile's x- and y-neighbours are streamed at the same z at the same time and each halo
// re-read is an L2 hit.  The remaining CTAs split the slab [lock_zm, nz) evenly.
struct CtaWork {
    int zb, len;
    int qb, qe;  // tile-planes: tiles * nz < 2^31 for any grid that fits the device
};

// Computed once per kernel by thread 0 (block_setup) and kept in shared memory: the split does
// not change between sweeps, and its 64-bit divisions would otherwise sit at the head of every
// sweep (a Taylor launch runs up to ~100 of them).
__shared__ CtaWork s_cw;

__device__ __forceinline__ CtaWork cta_work_compute(const SolveParams& p) {
    CtaWork w;
    const int64_t tiles = static_cast<int64_t>((p.op.nx + kTmaTX - 1) / kTmaTX) * ((p.op.ny + kTmaTY - 1) / kTmaTY);
    const int64_t b = vcta(), G = vncta();
    const int k = p.lock_groups;
    if (k > 0 && G >= k * tiles) {
        const int64_t kP = k * tiles;
        if (b < kP) {
            const int j = static_cast<int>(b / tiles);
            w.zb = j * p.lock_zm / k;
            w.len = (j + 1) * p.lock_zm / k - w.zb;
            w.qb = static_cast<int>((b % tiles) * w.len);
            w.qe = w.qb + w.len;
        } else {
            w.zb = p.lock_zm;
            w.len = p.op.nz - p.lock_zm;
            const int64_t qs = tiles * w.len, E = G - kP, e = b - kP;
            w.qb = static_cast<int>(e * qs / E);
            w.qe = static_cast<int>((e + 1) * qs / E);
        }
        if (w.len <= 0) w.len = 1, w.qb = w.qe = 0;
        return w;
    }
    w.zb = 0;
    w.len = p.op.nz;
    const int64_t Q = tiles * p.op.nz;
    w.qb = static_cast<int>(b * Q / G);
    w.qe = static_cast<int>((b + 1) * Q / G);
    return w;
}

__device__ __forceinline__ CtaWork cta_work() { return s_cw; }

// TMA z-slab sweep.  `seq` counts plane loads issued so far in this launch (identical in
// every thread); it fixes each ring slot's mbarrier phase parity.
template <bool kNeedF, bool kNeedB, class Body>
__device__ __forceinline__ void sweep_tma(const SolveParams& p, const Ring& ring, int xbuf, int fbuf, int bbuf,
                                          uint32_t& seq, const double* s_wtab, Body&& body) {
    const StencilOp& op = p.op;
    // read once (the ensemble kernels' p lives in global memory: see sweep2_tma)
    const int op_nx = op.nx, op_ny = op.ny, op_nz = op.nz;
    const int64_t op_sy = op.sy, op_sz = op.sz;
    const int tid = threadIdx.x;
    const int lane = tid & 31, row = tid >> 5;
    const int tiles_x = (op_nx + kTmaTX - 1) / kTmaTX;
    const int tiles_y = (op_ny + kTmaTY - 1) / kTmaTY;
    const CtaWork cw = cta_work();
    const int q_begin = cw.qb, q_end = cw.qe;
    constexpr uint32_t kOwnBytes = kLBytes + (kNeedF ? kOBytes : 0) + (kNeedB ? kOBytes : 0);
    constexpr uint32_t kHaloBytes = (kTmaTY + 2) * kXPitch * 8;
    if (tid == 0) fence_proxy_async_global();  // generic writes before this sweep -> TMA reads
    const uint64_t pol_labels = l2_policy_evict_last();  // labels stay in L2 (see sweep2_tma)

    for (int q = q_begin; q < q_end;) {
        // (unsigned 32-bit divisions: the operands are non-negative and small)
        const unsigned tile = static_cast<unsigned>(q) / static_cast<unsigned>(cw.len);
        const int z0 = cw.zb + (q - static_cast<int>(tile) * cw.len);
        const int z1 = min(cw.zb + cw.len, z0 + (q_end - q));
        q += z1 - z0;
        const unsigned ty = tile / static_cast<unsigned>(tiles_x);
        const int x0 = static_cast<int>(tile - ty * tiles_x) * kTmaTX;
        const int y0 = static_cast<int>(ty) * kTmaTY;
        const uint32_t base = seq;
        const int np = z1 - z0 + 2;  // planes z0-1 .. z1

        auto issue = [&](int pl) {
            const uint32_t sq = base + static_cast<uint32_t>(pl - (z0 - 1));
            const int slot = static_cast<int>(sq % kTmaStages);
            uint64_t* bar = ring.bar + slot;
            const bool own = pl >= z0 && pl < z1;
            mbar_arrive_expect_tx(bar, kHaloBytes + (own ? kOwnBytes : 0));
            tma_load_3d(ring.x(slot), &p.xmap[xbuf], x0 - kXHalo, y0 - 1, pl, bar);
            if (own) {
                if (kNeedF) tma_load_3d(ring.f(slot), &p.omap[fbuf], x0, y0, pl, bar);
                if (kNeedB) tma_load_3d(ring.b(slot), &p.omap[bbuf], x0, y0, pl, bar);
                tma_load_3d_hint(ring.l(slot), &p.lmap, x0, y0, pl, bar, pol_labels);
            }
        };
        auto slot_of = [&](int pl) { return static_cast<int>((base + static_cast<uint32_t>(pl - (z0 - 1))) % kTmaStages); };
        auto wait_plane = [&](int pl) {
            const uint32_t sq = base + static_cast<uint32_t>(pl - (z0 - 1));
            mbar_wait(ring.bar + sq % kTmaStages, (sq / kTmaStages) & 1u);
        };

        if (tid == 0) {
            const int pre = min(kTmaStages, np);
            for (int k = 0; k < pre; ++k) issue(z0 - 1 + k);
        }

        // this thread's two points of the tile: two columns of row `row` (64-wide tiles), or
        // rows `row` and `row + 16` of one column (32-wide tiles)
        static_assert(kTmaTX * kTmaTY == 2 * kSolveThreads, "two points per thread");
        constexpr bool kCols = kTmaTX == 64;
        int lxs[2], rws[2], ii[2], jj[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            lxs[c] = kCols ? lane + 32 * c : lane;
            rws[c] = kCols ? row : row + (kSolveThreads / 32) * c;
            ii[c] = x0 + lxs[c];
            jj[c] = y0 + rws[c];
        }
        double xm[2], xc[2];
        wait_plane(z0 - 1);
        wait_plane(z0);
        {
            const double* Xm = ring.x(slot_of(z0 - 1));
            const double* Xc = ring.x(slot_of(z0));
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                xm[c] = Xm[(rws[c] + 1) * kXPitch + lxs[c] + kXHalo];
                xc[c] = Xc[(rws[c] + 1) * kXPitch + lxs[c] + kXHalo];
            }
        }
        for (int z = z0; z < z1; ++z) {
            wait_plane(z + 1);
            const int sc = slot_of(z), sp = slot_of(z + 1);
            const double* Xc = ring.x(sc);
            const double* Xp = ring.x(sp);
            const double* Fo = ring.f(sc);
            const double* Bo = ring.b(sc);
            const uint8_t* Lo = ring.l(sc);
            const bool hz0 = z > 0, hz1 = z < op_nz - 1;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int lx = lxs[c], rw = rws[c];
                const int i = ii[c], j = jj[c];
                const bool hy0 = j > 0, hy1 = j < op_ny - 1;
                const double xp = Xp[(rw + 1) * kXPitch + lx + kXHalo];
                if (i < op_nx && j < op_ny) {
                    const double xym = Xc[rw * kXPitch + lx + kXHalo];
                    const double xyp = Xc[(rw + 2) * kXPitch + lx + kXHalo];
                    const double xxm = Xc[(rw + 1) * kXPitch + lx + kXHalo - 1];
                    const double xxp = Xc[(rw + 1) * kXPitch + lx + kXHalo + 1];
                    const int o = rw * kTmaTX + lx;
                    RowCoef rc;
                    rc.w = s_wtab[Lo[o]];
                    rc.live = rc.w != 0.0;
                    const int cnt = (i > 0) + (i < op_nx - 1) + hy0 + hy1 + hz0 + hz1;
                    const double acc = row_apply(rc, cnt, xm[c], xym, xxm, xc[c], xxp, xyp, xp);
                    const int64_t v = i + static_cast<int64_t>(j) * op_sy + static_cast<int64_t>(z) * op_sz;
                    body(v, acc, xc[c], kNeedF ? Fo[o] : 0.0, kNeedB ? Bo[o] : 0.0);
                }
                xm[c] = xc[c];
                xc[c] = xp;
            }
            __syncthreads();  // every thread is done with plane z-1's slot
            if (tid == 0) {
                const int nxt = z - 1 + kTmaStages;
                if (nxt <= z1) issue(nxt);
            }
        }
        seq = base + static_cast<uint32_t>(np);
    }
    fence_proxy_async_global();  // this thread's generic writes -> later TMA reads
}

// ------------------------------------------------------------------------------------------
// Two-term fused TMA sweep (temporal blocking)
// ------------------------------------------------------------------------------------------
// One pass over HBM computes two consecutive Taylor terms (expact.cpp:81-95 twice):
//   T1 = c1 * (A~ X)          on the tile plus a one-voxel halo, per plane, into a 3-plane
//                             shared ring (OOB points hold 0.0, i.e. missing neighbours)
//   T2 = c2 * (A T1)          on the tile
//   F1 = Fprev + T1, F2 = F1 + T2  (the reference's f += term, same operations, same order)
// and writes T2 and F1; F2 = F1 + T2 stays implicit (recomputed bit-exactly by its consumer).
// The four maxima |T1|, |F1|, |T2|, |F2| feed the two termination tests.
//
// Kinds:   first-zero    stage 0 of the bordered action: T1 = c1*(0 + b/gamma), Fprev = 0
//          first-border  stage >= 1: X = f, T1 = c1*(A f + b/gamma), Fprev = f
//          first-plain   expmv stage start: X = f, T1 = c1*(A f), Fprev = f
//          next          X = T_j, Fprev = F_{j-1} + T_j (state kept as (T_j, F_{j-1}))
enum Fused2Kind { k2FirstZero = 0, k2FirstBorder = 1, k2FirstPlain = 2, k2Next = 3 };

// Two-term ring layouts.  Plain: slots of [X halo-2 | F own or b/gamma halo-1 | labels].
// Implicit X (kImp, a stage's first sweep from f = F + T): [F halo-2, combined in place into
// X | T halo-2 | b/gamma halo-1 | labels], fewer stages.  T1 planes follow the slots.
template <int kSt, bool kImpl>
struct Ring2T {
    static constexpr int kStages = kSt;
    static constexpr bool kImp = kImpl;
    static constexpr int kSlot = kImpl ? k2ISlotBytes : k2SlotBytes;
    static constexpr int kFBOff = kImpl ? 2 * k2XBytes : k2XBytes;
    unsigned char* base;
    uint64_t* bar;
    __device__ double* x(int s) const { return reinterpret_cast<double*>(base + s * kSlot); }
    __device__ double* t(int s) const { return reinterpret_cast<double*>(base + s * kSlot + k2XBytes); }
    __device__ double* f(int s) const { return reinterpret_cast<double*>(base + s * kSlot + kFBOff); }
    __device__ double* b(int s) const { return reinterpret_cast<double*>(base + s * kSlot + kFBOff); }
    __device__ uint8_t* l(int s) const { return base + s * kSlot + kFBOff + k2FBBytes; }
    __device__ double* t1(int q) const { return reinterpret_cast<double*>(base + kSt * kSlot + q * kT1Bytes); }
};
using Ring2 = Ring2T<k2Stages, false>;
using Ring2I = Ring2T<k2IStages, true>;

// kSkipOut: planes past the grid skip their (all-zero) T1 stencil work -- worth it on thin
// grids (2-D: two of every three T1 planes), a separate instantiation so the deep-grid
// kernel's code is unchanged.
//
// Implicit X (R::kImp): the stage's start vector f = F[xbuf] + T[fbuf] is never stored: each
// plane's two halo tiles land by TMA and are summed in place (the same __dadd_rn as the
// reference's f += term), each thread its own points, its T1-ring point and one outer-halo
// point, so nothing is read before its own thread wrote it until the plane's barrier.
template <int KIND, bool kSkipOut = false, bool kExact = false, class R = Ring2>
__device__ __forceinline__ void sweep2_tma(const SolveParams& p, const R& ring, int xbuf, int fbuf, int bbuf,
                                           double c1, double c2, double* outT, double* outF, double (&mx)[5],
                                           uint32_t& seq, uint32_t& phase_mask, const double* s_wtab) {
    // Register-blocked layout: thread t owns column xl = t % kTmaTX and rows ry0 = 2*(t/kTmaTX),
    // ry0+1 of the tile for the whole z-march, so its z-1/z/z+1 values of X and T1 and its own
    // y-neighbour live in registers; x-neighbours and the outer y-neighbours come from shared
    // memory.  The halo-ring points of T1 (no corners; 128 with 32 x 32 tiles) are computed by
    // the first kRing threads from shared memory.
    // All per-thread shared-memory offsets are fixed per tile; ring slots rotate by increment and
    // barrier parities are tracked in a bit mask (identical in every thread).
    constexpr bool needX = KIND != k2FirstZero;
    constexpr bool kImp = R::kImp;
    constexpr int kSt = R::kStages;
    static_assert(!kImp || KIND == k2FirstBorder || KIND == k2FirstPlain, "implicit X only starts a stage");
    constexpr bool needF = KIND == k2Next;
    constexpr bool needB = KIND == k2FirstZero || KIND == k2FirstBorder;
    constexpr uint32_t kXTx = k2XRows * kXPitch * 8;
    constexpr uint32_t kBTx = k2BRows * kXPitch * 8;
    constexpr uint32_t kLTx = (kTmaTY + 2) * kLPitch;
    // T1 halo ring: rows -1 and kTmaTY over the tile's columns, columns -1 and kTmaTX over its
    // rows -- phase B's 5-point in-plane stencil never reads the four corners.  128 points with
    // 32 x 32 tiles: warps 0-3, one per SM sub-partition (160 with 64 x 16: warps 0-4).
    constexpr int kRing = 2 * kTmaTX + 2 * kTmaTY;
    // The thread that issues the TMA loads: lane 0 of warp 9 (a warp without ring points, on
    // a scheduler with one ring warp), not thread 0 of ring warp 0: +0.7% at C4 (measured
    // against warps 0 and 15).
    constexpr int kIssuer = kSolveThreads / 2 + 32;
    static_assert(kIssuer >= kRing && kIssuer < kSolveThreads, "the issuer has no ring point");
    const StencilOp& op = p.op;
    // The grid extents and strides the z-loop uses, read once: in the ensemble kernel p lives in
    // global memory and the compiler must otherwise reload them after every store (five LDG per
    // plane at the head of the dependency chains; long_scoreboard 20% of its stall samples).
    const int op_nz = op.nz;
    const int64_t op_sy = op.sy, op_sz = op.sz;
    // dead-row selects only in the exact instantiation (row_apply_ns)
    auto rowap = [](double w, bool live, double negcnt, double a, double b, double c, double d, double e, double f,
                    double g) {
        if constexpr (kExact) return row_apply_nc(w, live, negcnt, a, b, c, d, e, f, g);
        else return row_apply_ns(w, negcnt, a, b, c, d, e, f, g);
    };
    const int tid = threadIdx.x;
    const int xl = tid & (kTmaTX - 1);
    const int ry0 = 2 * (tid / kTmaTX);
    const int oX = (ry0 + 2) * kXPitch + xl + kXHalo;   // own row 0 in the X halo-2 tile
    const int oT = oX - kXPitch - 1;                    // own row 0 in a T1 plane (same pitch)
    const int oL = (ry0 + 1) * kLPitch + xl + kLHaloX;  // own row 0 in the label tile
    const int oB = oX - kXPitch;                        // own row 0 in the b/gamma tile
    const int oF = ry0 * kTmaTX + xl;                   // own row 0 in the F tile
    // this thread's ring point (rows -1 and kTmaTY, then columns -1 and kTmaTX); ring coordinates
    // (rr, rc) count from row -1 / column -1
    const bool ringer = tid < kRing;
    int rr = 0, rc = 0;
    if (ringer) {
        if (tid < 2 * kTmaTX) {
            rr = tid < kTmaTX ? 0 : kTmaTY + 1;
            rc = (tid & (kTmaTX - 1)) + 1;
        } else {
            const int e = tid - 2 * kTmaTX;
            rr = 1 + (e >> 1);
            rc = (e & 1) ? kTmaTX + 1 : 0;
        }
    }
    const int rX = (rr + 1) * kXPitch + rc + 1, rT = rX - kXPitch - 1, rL = rr * kLPitch + rc + kLHaloX - 1,
              rB = rX - kXPitch;

    const int tiles_x = (op.nx + kTmaTX - 1) / kTmaTX;
    const int tiles_y = (op.ny + kTmaTY - 1) / kTmaTY;
    const CtaWork cw = cta_work();
    const int q_begin = cw.qb, q_end = cw.qe;
    if (tid == kIssuer) fence_proxy_async_global();
    const uint64_t pol_labels = l2_policy_evict_last();
    unsigned mk[4] = {0u, 0u, 0u, 0u};  // bounding maxima (kExact == false): see max_key

    for (int q = q_begin; q < q_end;) {
        // (unsigned 32-bit divisions: the operands are non-negative and small)
        const unsigned tile = static_cast<unsigned>(q) / static_cast<unsigned>(cw.len);
        const int z0 = cw.zb + (q - static_cast<int>(tile) * cw.len);
        const int z1 = min(cw.zb + cw.len, z0 + (q_end - q));
        q += z1 - z0;
        const unsigned ty = tile / static_cast<unsigned>(tiles_x);
        const int x0 = static_cast<int>(tile - ty * tiles_x) * kTmaTX;
        const int y0 = static_cast<int>(ty) * kTmaTY;
        const uint32_t base = seq;
        const int pfirst = z0 - 2, plast = z1 + 1;  // planes loaded
        const int np = plast - pfirst + 1;

        // Static slots (kStatic: six stages, the z-loop unrolled by six): every segment starts at
        // slot 0 -- the ring is empty between segments, every issued plane has been waited for --
        // so plane pfirst + k sits in slot k % 6, a compile-time index inside the unrolled loop, and
        // every shared-memory address of the loop is a per-thread base plus an immediate.
        constexpr bool kStatic = kSt == 6;
        auto issue = [&](int pl) {  // the issuer only
            const int slot = kStatic ? (pl - pfirst) % kSt
                                     : static_cast<int>((base + static_cast<uint32_t>(pl - pfirst)) % kSt);
            uint64_t* bar = ring.bar + slot;
            const bool ownF = needF && pl >= z0 && pl < z1;
            const bool haloB = needB && pl >= z0 - 1 && pl <= z1;
            const bool haloL = pl >= z0 - 1 && pl <= z1;
            const uint32_t bytes = (needX ? kXTx : 0) + (kImp ? kXTx : 0) + (ownF ? kOBytes : 0) + (haloB ? kBTx : 0) +
                                   (haloL ? kLTx : 0);
            mbar_arrive_expect_tx(bar, bytes);
            if (needX) tma_load_3d(ring.x(slot), &p.x2map[xbuf], x0 - kXHalo, y0 - 2, pl, bar);
            if (kImp) tma_load_3d(ring.t(slot), &p.x2map[fbuf], x0 - kXHalo, y0 - 2, pl, bar);
            if (ownF) tma_load_3d(ring.f(slot), &p.omap[fbuf], x0, y0, pl, bar);
            if (haloB) tma_load_3d(ring.b(slot), &p.xmap[bbuf], x0 - kXHalo, y0 - 1, pl, bar);
            // labels (1 B/voxel, 16.8 MB at 256^3) are re-read by every sweep: keep them in L2
            // ahead of the streamed fp64 vectors
            if (haloL) tma_load_3d_hint(ring.l(slot), &p.l2map, x0 - kLHaloX, y0 - 1, pl, bar, pol_labels);
        };
        auto wait_slot = [&](int slot) {
            mbar_wait(ring.bar + slot, (phase_mask >> slot) & 1u);
            phase_mask ^= 1u << slot;
        };
        auto next_slot = [](int s) { return s + 1 == kSt ? 0 : s + 1; };

        if (tid == kIssuer) {
            const int pre = min(kSt, np);
            for (int k = 0; k < pre; ++k) issue(pfirst + k);
        }

        // per-segment geometry
        const int gx = x0 + xl, gy0 = y0 + ry0;
        const bool inx = gx < op.nx;
        const bool in0 = inx && gy0 < op.ny, in1 = inx && gy0 + 1 < op.ny;
        const int cxy = (gx > 0) + (gx < op.nx - 1);
        const double ncxy0 = -static_cast<double>(cxy + (gy0 > 0) + (gy0 < op.ny - 1));
        const double ncxy1 = -static_cast<double>(cxy + (gy0 + 1 > 0) + (gy0 + 1 < op.ny - 1));
        const int rgx = x0 - 1 + rc, rgy = y0 - 1 + rr;
        const double rncxy = -static_cast<double>((rgx > 0) + (rgx < op.nx - 1) + (rgy > 0) + (rgy < op.ny - 1));
        const int64_t v0 = gx + static_cast<int64_t>(gy0) * op_sy;

        // Phase A: T1 of plane pl.  sm/sc/sp: ring slots of planes pl-1, pl, pl+1.
        // xm/xc/xp: own rows' X at pl-1, pl, pl+1.  Writes T1's shared plane (pl & 1).
        // T1 shared planes rotate per segment: plane pl lives in slot (pl - z0 + 1) % 3, a
        // compile-time index inside the unrolled loop
        auto phaseA = [&](int pl, int tslot, int sm_, int sc_, int sp_, const double (&xm)[2], const double (&xc)[2],
                          const double (&xp)[2], double (&t1)[2], double (&lw)[2]) {
            double* T1 = ring.t1(tslot);
            if (kSkipOut && static_cast<unsigned>(pl) >= static_cast<unsigned>(op_nz)) {
                // a plane past the grid (z = -1 or nz): T1 is all zero there -- no stencil work
                // (2-D grids would otherwise compute three planes per useful one)
                t1[0] = t1[1] = 0.0;
                T1[oT] = 0.0;
                T1[oT + kT1Pitch] = 0.0;
                if (ringer) T1[rT] = 0.0;
                return;
            }
            const double dhz = static_cast<double>((pl > 0) + (pl < op_nz - 1));
            const double* Xc = ring.x(sc_);
            const uint8_t* L = ring.l(sc_);
            const double* B = ring.b(sc_);
            const double w0 = s_wtab[L[oL]], w1 = s_wtab[L[oL + kLPitch]];
            lw[0] = w0;
            lw[1] = w1;
            double s0, s1;
            if (KIND == k2FirstZero) {
                s0 = __dadd_rn(0.0, B[oB]);
                s1 = __dadd_rn(0.0, B[oB + kXPitch]);
            } else {
                const double xr0m = Xc[oX - 1], xr0p = Xc[oX + 1], xr1m = Xc[oX + kXPitch - 1], xr1p = Xc[oX + kXPitch + 1];
                const double xym0 = Xc[oX - kXPitch], xyp1 = Xc[oX + 2 * kXPitch];
                s0 = rowap(w0, w0 != 0.0, __dsub_rn(ncxy0, dhz), xm[0], xym0, xr0m, xc[0], xr0p, xc[1], xp[0]);
                s1 = rowap(w1, w1 != 0.0, __dsub_rn(ncxy1, dhz), xm[1], xc[0], xr1m, xc[1], xr1p, xyp1, xp[1]);
                if (KIND == k2FirstBorder) {
                    s0 = __dadd_rn(s0, B[oB]);
                    s1 = __dadd_rn(s1, B[oB + kXPitch]);
                }
            }
            // Outside the grid (planes -1 / nz, rows or columns past the edge) TMA zero-fills
            // the labels, and palette index 0 is always D = 0: the row is dead, s = 0 and T1 is
            // a signed zero, which as a neighbour adds nothing (accumulators start at +0.0).
            const double v0_ = __dmul_rn(c1, s0);
            const double v1_ = __dmul_rn(c1, s1);
            t1[0] = v0_;
            t1[1] = v1_;
            T1[oT] = v0_;
            T1[oT + kT1Pitch] = v1_;
            if (ringer) {
                const double w = s_wtab[L[rL]];
                double sc;
                if (KIND == k2FirstZero) {
                    sc = __dadd_rn(0.0, B[rB]);
                } else {
                    const double* Xm = ring.x(sm_);
                    const double* Xp = ring.x(sp_);
                    sc = rowap(w, w != 0.0, __dsub_rn(rncxy, dhz), Xm[rX], Xc[rX - kXPitch], Xc[rX - 1], Xc[rX],
                                      Xc[rX + 1], Xc[rX + kXPitch], Xp[rX]);
                    if (KIND == k2FirstBorder) sc = __dadd_rn(sc, B[rB]);
                }
                T1[rT] = __dmul_rn(c1, sc);
            }
        };

        // implicit X: X = F + T over plane slot s, this thread's points (see above); returns
        // the own rows' values
        auto combine = [&](int s, double (&xo)[2]) {
            double* Xs = ring.x(s);
            const double* Ts = ring.t(s);
            xo[0] = Xs[oX] = __dadd_rn(Xs[oX], Ts[oX]);
            xo[1] = Xs[oX + kXPitch] = __dadd_rn(Xs[oX + kXPitch], Ts[oX + kXPitch]);
            if (ringer) Xs[rX] = __dadd_rn(Xs[rX], Ts[rX]);
            // outer halo: X-tile rows 0 and k2XRows-1, then columns
            // 0 and kXPitch-1 of the rows between; then the four ring corners (row -1 / 16 x
            // column -1 / 64: not T1 ring points, but x-neighbours of the ring's end points);
            // threads from kRing on, wrapping if too few
            constexpr int kEdge = 2 * kXPitch + 2 * (kTmaTY + 2);
            constexpr int kOuter = kEdge + 4;
            for (int e = tid - kRing; e < kOuter; e += kSolveThreads - kRing) {
                if (e < 0) break;
                const int f = e - 2 * kXPitch;
                int o;
                if (e >= kEdge) {
                    const int k = e - kEdge;
                    o = ((k & 2) ? kTmaTY + 2 : 1) * kXPitch + ((k & 1) ? kTmaTX + 2 : 1);
                } else {
                    o = f < 0 ? (e < kXPitch ? e : (k2XRows - 1) * kXPitch + e - kXPitch)
                              : (1 + (f >> 1)) * kXPitch + ((f & 1) ? kXCols - 1 : 0);
                }
                Xs[o] = __dadd_rn(Xs[o], Ts[o]);
            }
            fence_proxy_async_shared();  // generic writes into a TMA slot before its next fill
        };

        const int s0 = kStatic ? 0 : static_cast<int>(base % kSt);  // slot of plane z0-2
        const int s1 = next_slot(s0), s2 = next_slot(s1), s3 = next_slot(s2);
        // prologue: T1 of planes z0-1 and z0
        wait_slot(s0);
        wait_slot(s1);
        wait_slot(s2);
        double xz[2] = {0.0, 0.0}, xa[2] = {0.0, 0.0}, xb[2] = {0.0, 0.0}, xn[2] = {0.0, 0.0};
        if constexpr (kImp) {
            wait_slot(s3);
            combine(s0, xz);
            combine(s1, xa);
            combine(s2, xb);
            combine(s3, xn);
            __syncthreads();
        } else if (needX) {
            const double* X0 = ring.x(s0);
            const double* X1 = ring.x(s1);
            const double* X2 = ring.x(s2);
            xz[0] = X0[oX];
            xz[1] = X0[oX + kXPitch];
            xa[0] = X1[oX];
            xa[1] = X1[oX + kXPitch];
            xb[0] = X2[oX];
            xb[1] = X2[oX + kXPitch];
        }
        // own T1 of planes z-2, z-1, z (relative to the loop's z); w unused here
        double tm1[2], t0[2], lwd[2];
        phaseA(z0 - 1, 0, s0, s1, s2, xz, xa, xb, tm1, lwd);
        if (!kImp) wait_slot(s3);
        if (needX && !kImp) {
            const double* X3 = ring.x(s3);
            xn[0] = X3[oX];
            xn[1] = X3[oX + kXPitch];
        }
        phaseA(z0, 1, s1, s2, s3, xa, xb, xn, t0, lwd);
        xa[0] = xb[0];
        xa[1] = xb[1];
        xb[0] = xn[0];
        xb[1] = xn[1];
        __syncthreads();
        if (tid == kIssuer) {
            if (pfirst + kSt <= plast) issue(pfirst + kSt);
            if (pfirst + 1 + kSt <= plast) issue(pfirst + 1 + kSt);
        }
        // Iteration z: phase A makes T1(z+1) (z < z1), phase B finishes plane z-1 (z > z0) --
        // independent work, so the two dependency chains overlap.  Register rings of three:
        // iteration z with r = (z - z0) % 3 finds X(z) in X3[r], X(z+1) in X3[r+1] and loads
        // X(z+2) into X3[r+2]; T1(z-1) in T3[r], T1(z) in T3[r+1], T1(z-2) in T3[r+2], which
        // phase A then overwrites with T1(z+1).  Unrolling by three makes every index static.
        double X3[3][2] = {{xa[0], xa[1]}, {xb[0], xb[1]}, {0.0, 0.0}};
        double T3[3][2] = {{tm1[0], tm1[1]}, {t0[0], t0[1]}, {0.0, 0.0}};
        int sM = s1, sA = s2, sB = s3, sC = next_slot(s3);  // slots of planes z-1, z, z+1, z+2
        double* pT = outT + v0 + static_cast<int64_t>(z0) * op_sz;
        double* pF = outF + v0 + static_cast<int64_t>(z0) * op_sz;
        auto iter = [&](int z, auto jconst) {
            constexpr int j = decltype(jconst)::value;  // (z - z0) % 6 (static slots) or % 3
            constexpr int r = j % 3;
            constexpr int r1 = (r + 1) % 3, r2 = (r + 2) % 3;
            if constexpr (kStatic) {
                sM = (j + 1) % 6;
                sA = (j + 2) % 6;
                sB = (j + 3) % 6;
                sC = (j + 4) % 6;
            }
            if (z > z0) {
                // Phase B: own voxels of plane zo = z-1 (T1 of zo-1, zo, zo+1 in T3[r2], T3[r], T3[r1])
                const int zo = z - 1;
                const double* T1s = ring.t1(r);  // plane zo = z - 1: slot (z - z0) % 3
                const uint8_t* L = ring.l(sM);
                const double w0 = s_wtab[L[oL]], w1 = s_wtab[L[oL + kLPitch]];
                const double dhz = static_cast<double>((zo > 0) + (zo < op_nz - 1));
                const double y0m = T1s[oT - kT1Pitch], y1p = T1s[oT + 2 * kT1Pitch];
                const double a0 = rowap(w0, w0 != 0.0, __dsub_rn(ncxy0, dhz), T3[r2][0], y0m, T1s[oT - 1],
                                               T3[r][0], T1s[oT + 1], T3[r][1], T3[r1][0]);
                const double a1 = rowap(w1, w1 != 0.0, __dsub_rn(ncxy1, dhz), T3[r2][1], T3[r][0],
                                               T1s[oT + kT1Pitch - 1], T3[r][1], T1s[oT + kT1Pitch + 1], y1p, T3[r1][1]);
                const double t20 = __dmul_rn(c2, a0), t21 = __dmul_rn(c2, a1);
                double fp0, fp1;
                if (KIND == k2FirstZero) {
                    fp0 = 0.0;
                    fp1 = 0.0;
                } else {
                    const double* XM = ring.x(sM);
                    const double xo0 = XM[oX], xo1 = XM[oX + kXPitch];
                    if constexpr (kExact) mx[4] = max_abs(max_abs(mx[4], xo0), xo1);
                    if (KIND == k2Next) {
                        const double* Fo = ring.f(sM);
                        fp0 = __dadd_rn(Fo[oF], xo0);
                        fp1 = __dadd_rn(Fo[oF + kTmaTX], xo1);
                    } else {
                        fp0 = xo0;
                        fp1 = xo1;
                    }
                }
                const double f10 = __dadd_rn(fp0, T3[r][0]), f11 = __dadd_rn(fp1, T3[r][1]);
                const double f20 = __dadd_rn(f10, t20), f21 = __dadd_rn(f11, t21);
                // The maxima drop NaN like std::max(m, |x|) (m is never NaN): expact.cpp:15-19.
                // They need no domain test: past the grid edge every input is zero-filled and the
                // row is dead (palette index 0), so T1, T2, F1 and F2 are signed zeros there.
                if constexpr (kExact) {
                    mx[0] = max_abs(max_abs(mx[0], T3[r][0]), T3[r][1]);
                    mx[1] = max_abs(max_abs(mx[1], f10), f11);
                    mx[2] = max_abs(max_abs(mx[2], t20), t21);
                    mx[3] = max_abs(max_abs(mx[3], f20), f21);
                } else {
                    mk[0] = max(max(mk[0], max_key(T3[r][0])), max_key(T3[r][1]));
                    mk[1] = max(max(mk[1], max_key(f10)), max_key(f11));
                    mk[2] = max(max(mk[2], max_key(t20)), max_key(t21));
                    mk[3] = max(max(mk[3], max_key(f20)), max_key(f21));
                }
                if (in0) {
                    pT[0] = t20;
                    pF[0] = f10;
                }
                if (in1) {
                    pT[op_sy] = t21;
                    pF[op_sy] = f11;
                }
                pT += op_sz;
                pF += op_sz;
            }
            if (z < z1) {
                wait_slot(sC);
                if constexpr (kImp) {
                    combine(sC, X3[r2]);
                } else if (needX) {
                    const double* XC = ring.x(sC);
                    X3[r2][0] = XC[oX];
                    X3[r2][1] = XC[oX + kXPitch];
                }
                double lwN[2];
                phaseA(z + 1, r2, sA, sB, sC, X3[r], X3[r1], X3[r2], T3[r2], lwN);
            }
            if constexpr (!kStatic) {
                sM = sA;
                sA = sB;
                sB = sC;
                sC = next_slot(sC);
            }
            __syncthreads();  // plane z-1's slot and T1(z-1)'s shared plane are free
            if (tid == kIssuer && z > z0) {
                const int nxt = z - 1 + kSt;
                if (nxt <= plast) issue(nxt);
            }
        };
        if constexpr (kStatic) {
            for (int zb = z0; zb <= z1; zb += 6) {
                iter(zb, std::integral_constant<int, 0>{});
                if (zb + 1 <= z1) iter(zb + 1, std::integral_constant<int, 1>{});
                if (zb + 2 <= z1) iter(zb + 2, std::integral_constant<int, 2>{});
                if (zb + 3 <= z1) iter(zb + 3, std::integral_constant<int, 3>{});
                if (zb + 4 <= z1) iter(zb + 4, std::integral_constant<int, 4>{});
                if (zb + 5 <= z1) iter(zb + 5, std::integral_constant<int, 5>{});
            }
        } else {
            for (int zb = z0; zb <= z1; zb += 3) {
                iter(zb, std::integral_constant<int, 0>{});
                if (zb + 1 <= z1) iter(zb + 1, std::integral_constant<int, 1>{});
                if (zb + 2 <= z1) iter(zb + 2, std::integral_constant<int, 2>{});
            }
        }
        seq = base + static_cast<uint32_t>(np);
    }
    if constexpr (!kExact) {
#pragma unroll
        for (int k = 0; k < 4; ++k) mx[k] = key_lower(mk[k]);
    }
    fence_proxy_async_global();
}

// ------------------------------------------------------------------------------------------
// Three-term fused TMA sweep (deeper temporal blocking)
// ------------------------------------------------------------------------------------------
// One pass over HBM computes three consecutive Taylor terms (expact.cpp:81-95 three times):
//   A: T1 = c1 * (A~ X)   on the tile plus a two-voxel ring   (4-plane shared ring)
//   B: T2 = c2 * (A T1)   on the tile plus a one-voxel ring   (3-plane shared ring)
//   C: T3 = c3 * (A T2)   on the tile;  F1 = Fprev + T1, F2 = F1 + T2, F3 = F2 + T3
// and writes T3 and F2 (F3 = F2 + T3 stays implicit; F1 is recomputed by a single-term
// sweep in the rare case a stage stops right after T1).  Iteration z runs A on plane z+1,
// B on plane z-1 and C on plane z-2: each reads only shared planes completed in earlier
// iterations (z-neighbours of its own points come from registers), so there is one barrier
// per plane.  Points outside the grid hold 0.0 in every ring (the missing neighbours).
struct Ring3 {
    unsigned char* base;
    uint64_t* barx;  // [k3XStages]
    uint64_t* barf;  // [k3FBStages]
    __device__ double* x(int s) const { return reinterpret_cast<double*>(base + s * k3XSlotBytes); }
    __device__ uint8_t* l(int s) const { return base + s * k3XSlotBytes + k3XBytes; }
    __device__ double* fb(int s) const {
        return reinterpret_cast<double*>(base + k3XStages * k3XSlotBytes + s * k3FBBytes);
    }
    __device__ double* t1(int q) const {
        return reinterpret_cast<double*>(base + k3XStages * k3XSlotBytes + k3FBStages * k3FBBytes + q * k3T1Bytes);
    }
    __device__ double* t2(int q) const {
        return reinterpret_cast<double*>(base + k3XStages * k3XSlotBytes + k3FBStages * k3FBBytes +
                                         k3T1Planes * k3T1Bytes + q * k3T2Bytes);
    }
};

template <int KIND>
__device__ __forceinline__ void sweep3_tma(const SolveParams& p, const Ring3& ring, int xbuf, int fbuf, double c1,
                                           double c2, double c3, double* outT, double* outF, double (&mx)[6],
                                           uint32_t& seqx, uint32_t& seqf, uint32_t& pmx, uint32_t& pmf,
                                           const double* s_wtab) {
    constexpr bool needX = KIND != k2FirstZero;
    constexpr bool needF = KIND == k2Next;
    constexpr bool needB = KIND == k2FirstZero || KIND == k2FirstBorder;
    constexpr uint32_t kXTx = k3XRows * k3XPitch * 8;
    constexpr uint32_t kLTx = k3LRows * kLPitch;
    constexpr uint32_t kBTx = k3BRows * k3XPitch * 8;
    constexpr int kARing = 2 * (kTmaTX + 4) * 2 + 4 * kTmaTY;  // 336 points of T1's two-voxel ring
    constexpr int kBRing = 2 * (kTmaTX + 2) + 2 * kTmaTY;      // 164 points of T2's one-voxel ring
    static_assert(KIND < 0 || kARing + kBRing <= kSolveThreads, "ring points need one thread each");
    const StencilOp& op = p.op;
    const int tid = threadIdx.x;
    const int xl = tid & (kTmaTX - 1);
    const int ry0 = 2 * (tid / kTmaTX);
    const int oX = (ry0 + 3) * k3XPitch + xl + k3XHaloX;
    const int oL = (ry0 + 2) * kLPitch + xl + kLHaloX;
    const int oB = (ry0 + 2) * k3XPitch + xl + k3XHaloX;
    const int oT1 = (ry0 + 2) * k3T1Pitch + xl + 2;
    const int oT2 = (ry0 + 1) * k3T2Pitch + xl + 1;
    const int oF = ry0 * kTmaTX + xl;
    // ring point of this thread: T1's ring for tid < 336, T2's ring for 336 <= tid < 500
    const bool aring = tid < kARing;
    const bool bring = !aring && tid < kARing + kBRing;
    int rr = 0, rc = 0;
    if (aring) {
        if (tid < 4 * (kTmaTX + 4)) {  // rows -2, -1, 16, 17 over columns -2 .. 65
            const int rowi = tid / (kTmaTX + 4);
            rr = rowi < 2 ? rowi - 2 : kTmaTY + rowi - 2;
            rc = tid % (kTmaTX + 4) - 2;
        } else {  // columns -2, -1, 64, 65 over rows 0 .. 15
            const int e = tid - 4 * (kTmaTX + 4);
            rr = e >> 2;
            const int k = e & 3;
            rc = k < 2 ? k - 2 : kTmaTX + k - 2;
        }
    } else if (bring) {
        const int b = tid - kARing;
        if (b < 2 * (kTmaTX + 2)) {  // rows -1 and 16 over columns -1 .. 64
            rr = b < kTmaTX + 2 ? -1 : kTmaTY;
            rc = b % (kTmaTX + 2) - 1;
        } else {  // columns -1 and 64 over rows 0 .. 15
            const int e = b - 2 * (kTmaTX + 2);
            rr = e >> 1;
            rc = (e & 1) ? kTmaTX : -1;
        }
    }
    const int aX = (rr + 3) * k3XPitch + rc + k3XHaloX;
    const int aL = (rr + 2) * kLPitch + rc + kLHaloX;
    const int aB = (rr + 2) * k3XPitch + rc + k3XHaloX;
    const int aT1 = (rr + 2) * k3T1Pitch + rc + 2;
    const int aT2 = (rr + 1) * k3T2Pitch + rc + 1;

    const int tiles_x = (op.nx + kTmaTX - 1) / kTmaTX;
    const int tiles_y = (op.ny + kTmaTY - 1) / kTmaTY;
    const CtaWork cw = cta_work();
    const int q_begin = cw.qb, q_end = cw.qe;
    if (tid == 0) fence_proxy_async_global();
    const uint64_t pol_labels = l2_policy_evict_last();  // labels stay in L2 (see sweep2_tma)

    for (int q = q_begin; q < q_end;) {
        // (unsigned 32-bit divisions: the operands are non-negative and small)
        const unsigned tile = static_cast<unsigned>(q) / static_cast<unsigned>(cw.len);
        const int z0 = cw.zb + (q - static_cast<int>(tile) * cw.len);
        const int z1 = min(cw.zb + cw.len, z0 + (q_end - q));
        q += z1 - z0;
        const unsigned ty = tile / static_cast<unsigned>(tiles_x);
        const int x0 = static_cast<int>(tile - ty * tiles_x) * kTmaTX;
        const int y0 = static_cast<int>(ty) * kTmaTY;
        const uint32_t basex = seqx, basef = seqf;
        const int pfirst = z0 - 3, plast = z1 + 2;  // X planes loaded
        const int fbfirst = needF ? z0 : z0 - 2;    // first F / b plane
        const int fblast = needF ? z1 - 1 : z1 + 1;
        const int nfb = (needF || needB) ? fblast - fbfirst + 1 : 0;

        auto issue_x = [&](int pl) {  // thread 0 only
            const int slot = static_cast<int>((basex + static_cast<uint32_t>(pl - pfirst)) % k3XStages);
            uint64_t* bar = ring.barx + slot;
            mbar_arrive_expect_tx(bar, (needX ? kXTx : 0) + kLTx);
            if (needX) tma_load_3d(ring.x(slot), &p.x3map[xbuf], x0 - k3XHaloX, y0 - 3, pl, bar);
            tma_load_3d_hint(ring.l(slot), &p.l3map, x0 - kLHaloX, y0 - 2, pl, bar, pol_labels);
        };
        auto issue_fb = [&](int pl) {  // thread 0 only
            const int slot = static_cast<int>((basef + static_cast<uint32_t>(pl - fbfirst)) % k3FBStages);
            uint64_t* bar = ring.barf + slot;
            if (needF) {
                mbar_arrive_expect_tx(bar, kOBytes);
                tma_load_3d(ring.fb(slot), &p.omap[fbuf], x0, y0, pl, bar);
            } else {
                mbar_arrive_expect_tx(bar, kBTx);
                tma_load_3d(ring.fb(slot), &p.b3map, x0 - k3XHaloX, y0 - 2, pl, bar);
            }
        };
        auto xslot = [&](int pl) { return static_cast<int>((basex + static_cast<uint32_t>(pl - pfirst)) % k3XStages); };
        auto fbslot = [&](int pl) {
            return static_cast<int>((basef + static_cast<uint32_t>(pl - fbfirst)) % k3FBStages);
        };
        auto wait_x = [&](int pl) {
            const int slot = xslot(pl);
            mbar_wait(ring.barx + slot, (pmx >> slot) & 1u);
            pmx ^= 1u << slot;
        };
        auto wait_fb = [&](int pl) {
            const int slot = fbslot(pl);
            mbar_wait(ring.barf + slot, (pmf >> slot) & 1u);
            pmf ^= 1u << slot;
        };

        if (tid == 0) {
            for (int k = 0; k < k3XStages && pfirst + k <= plast; ++k) issue_x(pfirst + k);
            for (int k = 0; k < k3FBStages && k < nfb; ++k) issue_fb(fbfirst + k);
        }

        // per-segment geometry (own points: column gx, rows gy0, gy0 + 1)
        const int gx = x0 + xl, gy0 = y0 + ry0;
        const bool inx = gx < op.nx;
        const bool in0 = inx && gy0 < op.ny, in1 = inx && gy0 + 1 < op.ny;
        const int cxy = (gx > 0) + (gx < op.nx - 1);
        const double ncxy0 = -static_cast<double>(cxy + (gy0 > 0) + (gy0 < op.ny - 1));
        const double ncxy1 = -static_cast<double>(cxy + (gy0 + 1 > 0) + (gy0 + 1 < op.ny - 1));
        const int rgx = x0 + rc, rgy = y0 + rr;
        const bool rin = (aring || bring) && rgx >= 0 && rgx < op.nx && rgy >= 0 && rgy < op.ny;
        const double rncxy = -static_cast<double>((rgx > 0) + (rgx < op.nx - 1) + (rgy > 0) + (rgy < op.ny - 1));
        const int64_t v0 = gx + static_cast<int64_t>(gy0) * op.sy;
        auto dhz = [&](int pl) { return static_cast<double>((pl > 0) + (pl < op.nz - 1)); };
        auto zin = [&](int pl) { return pl >= 0 && pl < op.nz; };

        // register rings (index = (plane - zb) & 3) of own values: X(z+1..z+2), T1(z-1..z+1),
        // T2(z-2..z-1); the oldest plane each phase needs is re-read from shared memory
        const int zb = z0 - 3;
        double Xr[4][2], T1r[4][2], T2r[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            Xr[k][0] = Xr[k][1] = 0.0;
            T1r[k][0] = T1r[k][1] = 0.0;
            T2r[k][0] = T2r[k][1] = 0.0;
        }
        wait_x(zb);
        wait_x(zb + 1);
        if (needX) {
            const double* X0 = ring.x(xslot(zb));
            const double* X1 = ring.x(xslot(zb + 1));
            Xr[0][0] = X0[oX];
            Xr[0][1] = X0[oX + k3XPitch];
            Xr[1][0] = X1[oX];
            Xr[1][1] = X1[oX + k3XPitch];
        }
        double* pT = outT + v0 + static_cast<int64_t>(z0) * op.sz;
        double* pF = outF + v0 + static_cast<int64_t>(z0) * op.sz;

        auto iter = [&](int z, auto rconst) {
            constexpr int r = decltype(rconst)::value;
            constexpr int r1 = (r + 1) & 3, r2 = (r + 2) & 3, r3 = (r + 3) & 3;
            // ---- A: T1 of plane pa = z + 1 (X of z, z+1, z+2 in Xr[r], Xr[r1], Xr[r2]) ----
            if (z <= z1) {
                const int pa = z + 1;
                wait_x(z + 2);
                const int sm_ = xslot(z), sc_ = xslot(pa), sp_ = xslot(z + 2);
                const double* Xc = ring.x(sc_);
                double xz0 = 0.0, xz1 = 0.0;  // own X(z): the ring's oldest plane, from shared memory
                if (needX) {
                    const double* Xp = ring.x(sp_);
                    Xr[r2][0] = Xp[oX];
                    Xr[r2][1] = Xp[oX + k3XPitch];
                    const double* Xm = ring.x(sm_);
                    xz0 = Xm[oX];
                    xz1 = Xm[oX + k3XPitch];
                }
                const double* B = nullptr;
                if (needB) {
                    wait_fb(pa);
                    B = ring.fb(fbslot(pa));
                }
                const uint8_t* L = ring.l(sc_);
                const bool za = zin(pa);
                const double dz = dhz(pa);
                const double w0 = s_wtab[L[oL]], w1 = s_wtab[L[oL + kLPitch]];
                double s0, s1;
                if (KIND == k2FirstZero) {
                    s0 = __dadd_rn(0.0, B[oB]);
                    s1 = __dadd_rn(0.0, B[oB + k3XPitch]);
                } else {
                    s0 = row_apply_nc(w0, w0 != 0.0, __dsub_rn(ncxy0, dz), xz0, Xc[oX - k3XPitch], Xc[oX - 1],
                                      Xr[r1][0], Xc[oX + 1], Xr[r1][1], Xr[r2][0]);
                    s1 = row_apply_nc(w1, w1 != 0.0, __dsub_rn(ncxy1, dz), xz1, Xr[r1][0],
                                      Xc[oX + k3XPitch - 1], Xr[r1][1], Xc[oX + k3XPitch + 1], Xc[oX + 2 * k3XPitch],
                                      Xr[r2][1]);
                    if (KIND == k2FirstBorder) {
                        s0 = __dadd_rn(s0, B[oB]);
                        s1 = __dadd_rn(s1, B[oB + k3XPitch]);
                    }
                }
                const double t0v = (za && in0) ? __dmul_rn(c1, s0) : 0.0;
                const double t1v = (za && in1) ? __dmul_rn(c1, s1) : 0.0;
                T1r[r1][0] = t0v;
                T1r[r1][1] = t1v;
                double* T1 = ring.t1(pa & 3);
                T1[oT1] = t0v;
                T1[oT1 + k3T1Pitch] = t1v;
                if (aring) {
                    const double w = s_wtab[L[aL]];
                    double sc;
                    if (KIND == k2FirstZero) {
                        sc = __dadd_rn(0.0, B[aB]);
                    } else {
                        const double* Xm = ring.x(sm_);
                        const double* Xp = ring.x(sp_);
                        sc = row_apply_nc(w, w != 0.0, __dsub_rn(rncxy, dz), Xm[aX], Xc[aX - k3XPitch], Xc[aX - 1],
                                          Xc[aX], Xc[aX + 1], Xc[aX + k3XPitch], Xp[aX]);
                        if (KIND == k2FirstBorder) sc = __dadd_rn(sc, B[aB]);
                    }
                    T1[aT1] = (za && rin) ? __dmul_rn(c1, sc) : 0.0;
                }
            }
            // ---- B: T2 of plane pb = z - 1 (own T1 of z-2, z-1, z in T1r[r2], T1r[r3], T1r[r]) ----
            if (z >= z0) {
                const int pb = z - 1;
                const double* T1m = ring.t1((pb + 3) & 3);
                const double* T1c = ring.t1(pb & 3);
                const double* T1p = ring.t1((pb + 1) & 3);
                const uint8_t* L = ring.l(xslot(pb));
                const bool zb_ = zin(pb);
                const double dz = dhz(pb);
                const double w0 = s_wtab[L[oL]], w1 = s_wtab[L[oL + kLPitch]];
                const double a0 = row_apply_nc(w0, w0 != 0.0, __dsub_rn(ncxy0, dz), T1m[oT1], T1c[oT1 - k3T1Pitch],
                                               T1c[oT1 - 1], T1r[r3][0], T1c[oT1 + 1], T1r[r3][1], T1r[r][0]);
                const double a1 = row_apply_nc(w1, w1 != 0.0, __dsub_rn(ncxy1, dz), T1m[oT1 + k3T1Pitch], T1r[r3][0],
                                               T1c[oT1 + k3T1Pitch - 1], T1r[r3][1], T1c[oT1 + k3T1Pitch + 1],
                                               T1c[oT1 + 2 * k3T1Pitch], T1r[r][1]);
                const double u0 = (zb_ && in0) ? __dmul_rn(c2, a0) : 0.0;
                const double u1 = (zb_ && in1) ? __dmul_rn(c2, a1) : 0.0;
                T2r[r3][0] = u0;
                T2r[r3][1] = u1;
                double* T2 = ring.t2((pb + 3) % 3);
                T2[oT2] = u0;
                T2[oT2 + k3T2Pitch] = u1;
                if (bring) {
                    const double w = s_wtab[L[aL]];
                    const double sc = row_apply_nc(w, w != 0.0, __dsub_rn(rncxy, dz), T1m[aT1], T1c[aT1 - k3T1Pitch],
                                                   T1c[aT1 - 1], T1c[aT1], T1c[aT1 + 1], T1c[aT1 + k3T1Pitch], T1p[aT1]);
                    T2[aT2] = (zb_ && rin) ? __dmul_rn(c2, sc) : 0.0;
                }
            }
            // ---- C: T3 of plane pc = z - 2 (own T2 of pc-1, pc, pc+1 in T2r[r1], T2r[r2], T2r[r3]) ----
            const bool runC = z >= z0 + 2;
            if (runC) {
                // reads T2's shared plane z-2 (written last iteration) and own T2 / T1 registers
                // only, so no barrier separates it from A and B
                const int pc = z - 2;
                const double* T2c = ring.t2((pc + 3) % 3);
                const double* T2m = ring.t2((pc + 2) % 3);
                const double* T1o = ring.t1(pc & 3);
                const uint8_t* L = ring.l(xslot(pc));
                const double dz = dhz(pc);
                const double w0 = s_wtab[L[oL]], w1 = s_wtab[L[oL + kLPitch]];
                const double b0 = row_apply_nc(w0, w0 != 0.0, __dsub_rn(ncxy0, dz), T2m[oT2], T2c[oT2 - k3T2Pitch],
                                               T2c[oT2 - 1], T2r[r2][0], T2c[oT2 + 1], T2r[r2][1], T2r[r3][0]);
                const double b1 = row_apply_nc(w1, w1 != 0.0, __dsub_rn(ncxy1, dz), T2m[oT2 + k3T2Pitch], T2r[r2][0],
                                               T2c[oT2 + k3T2Pitch - 1], T2r[r2][1], T2c[oT2 + k3T2Pitch + 1],
                                               T2c[oT2 + 2 * k3T2Pitch], T2r[r3][1]);
                const double t30 = __dmul_rn(c3, b0), t31 = __dmul_rn(c3, b1);
                double fp0, fp1;
                if (KIND == k2FirstZero) {
                    fp0 = 0.0;
                    fp1 = 0.0;
                } else {
                    const double* XC = ring.x(xslot(pc));
                    const double xo0 = XC[oX], xo1 = XC[oX + k3XPitch];
                    if (KIND == k2Next) {
                        wait_fb(pc);
                        const double* Fo = ring.fb(fbslot(pc));
                        fp0 = __dadd_rn(Fo[oF], xo0);
                        fp1 = __dadd_rn(Fo[oF + kTmaTX], xo1);
                    } else {
                        fp0 = xo0;
                        fp1 = xo1;
                    }
                }
                const double t10 = T1o[oT1], t11 = T1o[oT1 + k3T1Pitch];
                const double f10 = __dadd_rn(fp0, t10), f11 = __dadd_rn(fp1, t11);
                const double f20 = __dadd_rn(f10, T2r[r2][0]), f21 = __dadd_rn(f11, T2r[r2][1]);
                const double f30 = __dadd_rn(f20, t30), f31 = __dadd_rn(f21, t31);
                if (in0) {
                    pT[0] = t30;
                    pF[0] = f20;
                    mx[0] = max_abs(mx[0], t10);
                    mx[1] = max_abs(mx[1], f10);
                    mx[2] = max_abs(mx[2], T2r[r2][0]);
                    mx[3] = max_abs(mx[3], f20);
                    mx[4] = max_abs(mx[4], t30);
                    mx[5] = max_abs(mx[5], f30);
                }
                if (in1) {
                    pT[op.sy] = t31;
                    pF[op.sy] = f21;
                    mx[0] = max_abs(mx[0], t11);
                    mx[1] = max_abs(mx[1], f11);
                    mx[2] = max_abs(mx[2], T2r[r2][1]);
                    mx[3] = max_abs(mx[3], f21);
                    mx[4] = max_abs(mx[4], t31);
                    mx[5] = max_abs(mx[5], f31);
                }
                pT += op.sz;
                pF += op.sz;
            }
            __syncthreads();  // slots of plane z-2, T1(z-2)'s and T2(z-3)'s shared planes are free
            if (tid == 0) {
                const int freed = z - 2;  // X plane no longer read by any later iteration
                if (freed >= pfirst && freed + k3XStages <= plast) issue_x(freed + k3XStages);
                if (needF && runC && z - 2 + k3FBStages <= fblast) issue_fb(z - 2 + k3FBStages);
                if (needB && z <= z1 && z + 1 + k3FBStages <= fblast) issue_fb(z + 1 + k3FBStages);
            }
        };
        for (int zz = zb; zz <= z1 + 1; zz += 4) {
            iter(zz, std::integral_constant<int, 0>{});
            if (zz + 1 <= z1 + 1) iter(zz + 1, std::integral_constant<int, 1>{});
            if (zz + 2 <= z1 + 1) iter(zz + 2, std::integral_constant<int, 2>{});
            if (zz + 3 <= z1 + 1) iter(zz + 3, std::integral_constant<int, 3>{});
        }
        seqx = basex + static_cast<uint32_t>(plast - pfirst + 1);
        seqf = basef + static_cast<uint32_t>(nfb);
    }
    fence_proxy_async_global();
}

enum TermKind { kFirstZero, kFirstBorder, kFirstPlain, kNext };

// Per-block setup shared by the kernels: w table in shared memory, mbarriers for TMA.
template <class S>
__device__ __forceinline__ void block_setup(const SolveParams& p, S& sm, bool with_tma, bool reinit = false) {
    if (p.op.pal)
        for (int q = threadIdx.x; q < 256; q += blockDim.x) sm.wtab[q] = __ldg(p.op.wtab + q);
    if (with_tma && threadIdx.x == 0) {
        if (reinit) {  // every load on these barriers has completed and been waited for
            for (int s = 0; s < kTmaStages; ++s) mbar_inval(sm.bar1 + s);
            for (int s = 0; s < k2Stages; ++s) mbar_inval(sm.bar2 + s);
            for (int s = 0; s < k3XStages; ++s) mbar_inval(sm.bar3x + s);
            for (int s = 0; s < k3FBStages; ++s) mbar_inval(sm.bar3f + s);
        }
        for (int s = 0; s < kTmaStages; ++s) mbar_init(sm.bar1 + s, 1);
        for (int s = 0; s < k2Stages; ++s) mbar_init(sm.bar2 + s, 1);
        for (int s = 0; s < k3XStages; ++s) mbar_init(sm.bar3x + s, 1);
        for (int s = 0; s < k3FBStages; ++s) mbar_init(sm.bar3f + s, 1);
        mbar_fence_init();
        for (int b = 0; b < kNumBufs; ++b) tma_prefetch_desc(&p.xmap[b]);  // generic address: param or global
    }
    if (with_tma && threadIdx.x == 0) s_cw = cta_work_compute(p);
    __syncthreads();
}

__device__ __forceinline__ void trace_mark(const SolveParams& p, int tag) {
    if (p.trace && vcta() == 0 && threadIdx.x == 0) {
        const int k = atomicAdd(&p.ctrl->ntrace, 1);
        if (k < p.trace_cap) {
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            p.trace[2 * k] = static_cast<unsigned long long>(tag);
            p.trace[2 * k + 1] = tnow;
        }
    }
}

// Single-term stencil sweep dispatch (TMA ring or L1 fallback).
template <class S, class Body>
__device__ __forceinline__ void stencil_sweep(const SolveParams& p, S& sm, const Ring& ring, uint32_t& seq, int xb,
                                              int fb, int bb, Body&& body) {
    const bool nf = fb >= 0, nb = bb >= 0;
    if (p.op.csr_offs) {
        // generic CSR operator: grid-stride over rows
        const double* X = p.buf[xb];
        const double* F = nf ? p.buf[fb] : nullptr;
        const double* B = nb ? p.buf[bb] : nullptr;
        sweep_points(p.op, [&](int64_t v) {
            body(v, csr_row_apply(p.op, v, X), X[v], F ? F[v] : 0.0, B ? B[v] : 0.0);
        });
    } else if (p.use_tma) {
        if (nf && nb) sweep_tma<true, true>(p, ring, xb, fb, bb, seq, sm.wtab, body);
        else if (nf) sweep_tma<true, false>(p, ring, xb, fb, 0, seq, sm.wtab, body);
        else if (nb) sweep_tma<false, true>(p, ring, xb, 0, bb, seq, sm.wtab, body);
        else sweep_tma<false, false>(p, ring, xb, 0, 0, seq, sm.wtab, body);
    } else {
        sweep_l1(p.op, p.buf[xb], nf ? p.buf[fb] : nullptr, nb ? p.buf[bb] : nullptr, sm.wtab, body);
    }
}

// compute_metrics (integrator.cpp:65-89) accumulation: the sum in a fixed tree (the
// reference's serial sum differs in the last bits), max/min/front radius exactly.
struct MetricAcc {
    double sum = 0.0, mx = -INFINITY, mn = INFINITY, r2 = 0.0;
    __device__ __forceinline__ void add(const SolveParams& p, int64_t v, double u) {
        sum = __dadd_rn(sum, u);
        mx = nan_dropping_max(mx, u);
        mn = (u < mn) ? u : mn;
        if (u >= p.front_threshold) {
            const StencilOp& op = p.op;
            const int i = static_cast<int>(v % op.nx);
            const int j = static_cast<int>((v / op.nx) % op.ny);
            const int k = static_cast<int>(v / op.sz);
            const double dx = __dsub_rn(__dadd_rn(p.origin[0], __dmul_rn(static_cast<double>(i), p.h)), p.center[0]);
            const double dy = __dsub_rn(__dadd_rn(p.origin[1], __dmul_rn(static_cast<double>(j), p.h)), p.center[1]);
            const double dz = __dsub_rn(__dadd_rn(p.origin[2], __dmul_rn(static_cast<double>(k), p.h)), p.center[2]);
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            r2 = nan_dropping_max(r2, d2);
        }
    }
};

// Block-reduce the metric accumulators; the last block to finish (ticket) finalises node
// `node` from the per-block partials in a fixed order (deterministic for the launch size).
__device__ void metrics_commit(const SolveParams& p, Smem& sm, MetricAcc& a, int node) {
    double s[1] = {a.sum};
    block_reduce<1, false>(s, sm);
    const double mxw = warp_max(a.mx);
    double mnw = a.mn;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double q = __shfl_xor_sync(0xffffffffu, mnw, o);
        mnw = (q < mnw) ? q : mnw;
    }
    const double r2w = warp_max(a.r2);
    unsigned long long* ms = p.mslots;
    if ((threadIdx.x & 31) == 0) {
        atomicMax(ms + 0, ordered_key(mxw));
        atomicMin(ms + 1, ordered_key(mnw));
        if (r2w > 0.0) atomicMax(ms + 2, static_cast<unsigned long long>(__double_as_longlong(r2w)));
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        p.part_u[vcta()] = s[0];
        __threadfence();
        last = atomicAdd(&p.ctrl->ticket, 1u) == static_cast<unsigned>(vncta()) - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const double sum = grid_sum(p.part_u, vncta(), sm);
    if (threadIdx.x == 0) {
        const double cell = __dmul_rn(__dmul_rn(p.h, p.h), p.h);
        double* out = p.metrics + 4 * node;
        out[0] = __dmul_rn(cell, sum);
        out[1] = from_ordered_key(__ldcg(ms + 0));
        out[2] = from_ordered_key(__ldcg(ms + 1));
        out[3] = sqrt(__longlong_as_double(static_cast<long long>(__ldcg(ms + 2))));
        ms[0] = 0ull;
        ms[1] = ~0ull;
        ms[2] = 0ull;
        p.ctrl->ticket = 0u;
        __threadfence();
    }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// k_metrics: compute_metrics of the resident state (run node 0)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void metrics_body(const SolveParams& p) {
    __shared__ Smem sm;
    if (p.ctrl->status) return;
    const double* U = p.buf[kBufU];
    MetricAcc a;
    sweep_points(p.op, [&](int64_t v) { a.add(p, v, U[v]); });
    metrics_commit(p, sm, a, 0);
}

// ------------------------------------------------------------------------------------------
// K2 prep: RHS g = A u + rho u(1-u) and ||g||_1 partials (run); ||b||_1 / ||b||_inf
// partials (phi1v / expmv); y = A x (apply)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void prep_body(const SolveParams& p, int step) {
    __shared__ Smem sm;
    extern __shared__ __align__(128) unsigned char dyn[];
    if (p.ctrl->status) return;
    block_setup(p, sm, p.use_tma);
    trace_mark(p, kTrPrepIn);
    Ring ring{dyn, sm.bar1};
    uint32_t seq = 0;
    double* const G = p.buf[kBufG];
    double* const OUT = p.buf[kBufOut];
    if (p.mode == kModeApply) {
        stencil_sweep(p, sm, ring, seq, kBufG, -1, -1, [&](int64_t v, double acc, double, double, double) { OUT[v] = acc; });
        return;
    }
    double part = 0.0;
    if (p.mode == kModeRun) {
        // g = A u; g += rho*u*(1-u)   (integrator.cpp:54-57)
        stencil_sweep(p, sm, ring, seq, kBufU, -1, -1, [&](int64_t v, double acc, double u, double, double) {
            const double g = __dadd_rn(acc, __dmul_rn(__dmul_rn(p.rho, u), __dsub_rn(1.0, u)));
            G[v] = g;
            part = __dadd_rn(part, fabs(g));
        });
    } else if (p.mode == kModePhi1v) {
        sweep_points(p.op, [&](int64_t v) { part = __dadd_rn(part, fabs(G[v])); });  // expact.cpp:110
    } else {
        sweep_points(p.op, [&](int64_t v) { part = nan_dropping_max(part, fabs(G[v])); });  // expact.cpp:80
    }
    double s[1] = {part};
    if (p.mode == kModeExpmv) block_reduce<1, true>(s, sm);
    else block_reduce<1, false>(s, sm);
    if (threadIdx.x == 0) p.part_b[vcta()] = s[0];
    if (p.use_tma) fence_proxy_async_global();
}

// ------------------------------------------------------------------------------------------
// bordered column: ||b||_1, the degenerate branches, gamma and b/gamma + its column sum
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void border_body(const SolveParams& p, int prep_blocks, int step) {
    if (step < 0) step = __ldcg(&p.ctrl->step);  // graph replay: the step lives on the device
    __shared__ Smem sm;
    Ctrl* ctrl = p.ctrl;
    if (ctrl->status) return;
    trace_mark(p, kTrBorderIn);
    const bool leader = vcta() == 0 && threadIdx.x == 0;
    gs_step_info* info = (p.infos && leader) ? p.infos + step : nullptr;
    const double t = p.tau;
    double* const G = p.buf[kBufG];
    if (p.mode == kModeExpmv) {
        // prev = ||b||_inf (max of the partials: order-free)
        if (threadIdx.x == 0) {
            double m = 0.0;
            for (int b = 0; b < prep_blocks; ++b) m = nan_dropping_max(m, __ldcg(p.part_b + b));
            if (leader) {
                ctrl->prev0 = m;
                ctrl->branch = 0;
                ctrl->gamma = 0.0;
            }
        }
        if (info) {
            info->branch = 0;
            info->anorm = p.anorm;
        }
        return;
    }
    // expact.cpp:110: the reference's sequential sum (seqsum kernels) or, for A/B, a tree sum
    const double bnorm = p.seq_exact ? __ldcg(&ctrl->seq[0]) : grid_sum(p.part_b, prep_blocks, sm);
    int branch = 0;
    if (t == 0.0) branch = 1;                                  // expact.cpp:108
    else if (bnorm == 0.0) branch = 2;                         // expact.cpp:111
    else if (__dmul_rn(fabs(t), p.anorm) <= 1e-8) branch = 3;  // expact.cpp:114
    const double gamma = branch == 0 ? __ddiv_rn(bnorm, p.anorm) : 0.0;  // expact.cpp:126
    if (leader) {
        ctrl->bnorm = bnorm;
        ctrl->branch = branch;
        ctrl->gamma = gamma;
        ctrl->prev0 = 1.0;  // ||e_{n+1}||_inf
    }
    if (info) {
        info->s = info->m = 1;
        info->branch = branch;
        info->total_terms = 0;
        info->anorm = p.anorm;
        info->bnorm = bnorm;
        info->gamma = gamma;
        info->coln = info->norm_tA = 0.0;
    }
    if (branch != 0) return;
    // b/gamma in place where b != 0 (expact.cpp:137-138) and its column sum (sparse.cpp:36-38)
    double csum = 0.0;
    const int64_t tid = static_cast<int64_t>(vcta()) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(vncta()) * blockDim.x;
    const int64_t n = p.op.n;
    const int64_t n2 = n >> 1;
    double2* G2 = reinterpret_cast<double2*>(G);
    auto bg = [&](double b) { return (b != 0.0) ? __ddiv_rn(b, gamma) : 0.0; };
    constexpr int U = 4;
    for (int64_t i = tid; i < n2; i += U * stride) {
        double2 g[U];
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i + k * stride < n2) g[k] = G2[i + k * stride];
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i + k * stride < n2) {
                const double2 r = make_double2(bg(g[k].x), bg(g[k].y));
                G2[i + k * stride] = r;
                csum = __dadd_rn(csum, fabs(r.x));
                csum = __dadd_rn(csum, fabs(r.y));
            }
    }
    if ((n & 1) && tid == 0) {
        const double r = bg(G[n - 1]);
        G[n - 1] = r;
        csum = __dadd_rn(csum, fabs(r));
    }
    double s[1] = {csum};
    block_reduce<1, false>(s, sm);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        p.part_c[vcta()] = s[0];
        last = false;
        if (p.seq_exact) {  // the last CTA: does the tree column sum settle (s, m)?
            __threadfence();
            last = atomicAdd(&ctrl->border_ticket, 1u) == static_cast<unsigned>(vncta()) - 1;
        }
    }
    __syncthreads();
    if (last) {
        __threadfence();
        const double coln = grid_sum(p.part_c, vncta(), sm);
        if (threadIdx.x == 0) {
            ctrl->coln_need = seq::coln_settles(t, p.anorm, coln, n, p.rtab, kMaxDegree) ? 0 : 1;
            ctrl->border_ticket = 0u;
        }
    }
    if (p.use_tma) fence_proxy_async_global();
}

// ------------------------------------------------------------------------------------------
// K4 Taylor loop (cooperative, persistent): (s, m) on device, then the stages of fused
// two-term sweeps (TMA) or single-term sweeps (fallback) with the in-kernel termination
// test; grid barriers between terms.  The small-norm branch's stencil pass lives here too.
// ------------------------------------------------------------------------------------------
template <int FUSE, class GridBar>
__device__ __forceinline__ void taylor_body(const SolveParams& p, int border_blocks, int step, GridBar&& grid_bar,
                                            bool reinit) {
    if (step < 0) step = __ldcg(&p.ctrl->step);  // graph replay: the step lives on the device
    __shared__ SmemT sm;
    extern __shared__ __align__(128) unsigned char dyn[];
    Ctrl* ctrl = p.ctrl;
    if (ctrl->status) return;
    trace_mark(p, kTrTaylorIn);
    const StencilOp& op = p.op;
    if (threadIdx.x == 0) sm.red = reinterpret_cast<double (*)[6]>(dyn + kRedOffset);
    block_setup(p, sm, p.use_tma, reinit);
    Ring ring{dyn, sm.bar1};
    Ring2 ring2{dyn, sm.bar2};
    Ring2I ring2i{dyn, sm.bar2};
    Ring3 ring3{dyn, sm.bar3x, sm.bar3f};
    uint32_t seq = 0, seq2 = 0, pmask2 = 0, seq3x = 0, seq3f = 0, pm3x = 0, pm3f = 0;
    const bool leader = vcta() == 0 && threadIdx.x == 0;
    gs_step_info* info = (p.infos && leader) ? p.infos + step : nullptr;
    // Grid barrier; with TMA, first order this thread's generic global writes before any
    // later async-proxy (TMA) read of them.
    auto gsync = [&](int tag) {
        if (p.use_tma) fence_proxy_async_global();
        grid_bar();
        trace_mark(p, tag);
    };
    int round = 0;  // per-term max-reduction rounds (slot rotation, identical in every CTA)
    unsigned xround = p.xchg ? __ldcg(&ctrl->xround) : 0u;  // rounds of the maxima exchange (xchg_keys4)
    auto sync_round = [&](int tag) {
        gsync(tag);
        if (leader) {
            unsigned long long* z = p.slots + ((round + 2) % 3) * 8;
#pragma unroll
            for (int q = 0; q < 6; ++q) z[q] = 0ull;
        }
        ++round;
    };
    double* const G = p.buf[kBufG];
    const bool bordered = p.mode != kModeExpmv;
    const double t = p.tau;
    const int branch = __ldcg(&ctrl->branch);
    if (leader) {
        ctrl->fres = -1;
        ctrl->tres = -1;
    }
    if (branch != 0) {
        if (branch == 3) {
            // incr = b + 0.5*t*(A b)   (expact.cpp:117-121), into T0
            double* INC = p.buf[kBufT0];
            const double ht = __dmul_rn(0.5, t);
            stencil_sweep(p, sm, ring, seq, kBufG, -1, -1, [&](int64_t v, double acc, double b, double, double) {
                INC[v] = __dadd_rn(b, __dmul_rn(ht, acc));
            });
        }
        return;
    }

    // ------------------------------------------- bordered column norm and (s, m)
    const double gamma = __ldcg(&ctrl->gamma);
    double norm_tA;
    if (bordered) {
        // the exact (sequential) column sum when it was computed -- the step log asks for it, or
        // the tree sum's error bound straddles a (s, m) boundary -- else the tree sum, which
        // then provably selects the same (s, m) (seq::coln_settles)
        const bool exact = p.seq_exact && (p.infos || __ldcg(&ctrl->coln_need));
        const double coln = exact ? __ldcg(&ctrl->seq[1]) : grid_sum(p.part_c, border_blocks, sm);
        // bordered ||.||_1 = max over columns: A's columns, then column n (sparse.cpp:39-40)
        norm_tA = __dmul_rn(fabs(t), nan_dropping_max(p.anorm, coln));
        if (info) info->coln = coln;
    } else {
        norm_tA = __dmul_rn(fabs(t), p.anorm);
    }
    int s_st = 1, m_deg = 1;
    const int sel = select_params_dev(norm_tA, p.rtab, &s_st, &m_deg);
    if (info) {
        info->norm_tA = norm_tA;
        info->s = s_st;
        info->m = m_deg;
    }
    if (sel != GS_OK) {
        if (leader) {
            ctrl->status = sel;
            ctrl->detail = 1;  // select_params
        }
        return;  // uniform across CTAs
    }

    // ------------------------------------------------------------- K4: Taylor terms
    const double tau_s = __ddiv_rn(t, static_cast<double>(s_st));  // expact.cpp:73
    double prev = __ldcg(&ctrl->prev0);
    int64_t total_terms = 0;
    int reruns = 0;  // two-term sweeps re-run with exact maxima
    int fres = -1, tres = -1;  // stage result: F[fres] (+ T[tres] when tres >= 0, implicit)
    auto finite_or_fail = [&](double cur, double fnorm) {
        if (!isfinite(cur) || !isfinite(fnorm)) {  // expact.cpp:90-91
            if (leader) {
                ctrl->status = GS_ENUMERIC;
                ctrl->detail = 2;
            }
            return false;
        }
        return true;
    };
    // A stage starts from f: the previous stage's F[fres], materialising an implicit
    // F + T first (vectorised: two double2 loads per input in flight per thread).
    auto stage_start = [&](int stage) -> int {
        if (stage == 0) return bordered ? -1 : kBufG;
        if (tres < 0) return fres;
        const double* Fa = p.buf[fres];
        const double* Tb = p.buf[tres];
        const int fo = (fres == kBufF0) ? kBufF1 : kBufF0;
        double* Fw = p.buf[fo];
        const int64_t tid = static_cast<int64_t>(vcta()) * blockDim.x + threadIdx.x;
        const int64_t stride = static_cast<int64_t>(vncta()) * blockDim.x;
        const int64_t n2 = op.n >> 1;
        const double2* A2 = reinterpret_cast<const double2*>(Fa);
        const double2* B2 = reinterpret_cast<const double2*>(Tb);
        double2* W2 = reinterpret_cast<double2*>(Fw);
        for (int64_t i = tid; i < n2; i += 2 * stride) {
            const bool second = i + stride < n2;
            const double2 a0 = A2[i], b0 = B2[i];
            double2 a1 = make_double2(0.0, 0.0), b1 = a1;
            if (second) {
                a1 = A2[i + stride];
                b1 = B2[i + stride];
            }
            W2[i] = make_double2(__dadd_rn(a0.x, b0.x), __dadd_rn(a0.y, b0.y));
            if (second) W2[i + stride] = make_double2(__dadd_rn(a1.x, b1.x), __dadd_rn(a1.y, b1.y));
        }
        if ((op.n & 1) && tid == 0) Fw[op.n - 1] = __dadd_rn(Fa[op.n - 1], Tb[op.n - 1]);
        gsync(kTrFixup);
        return fo;
    };
    auto publish_max = [&](double* mx, int k, int tag) {
        if (threadIdx.x == 0) {
            unsigned long long* sl = p.slots + (round % 3) * 8;
            for (int q = 0; q < k; ++q)
                if (mx[q] > 0.0) atomicMax(sl + q, static_cast<unsigned long long>(__double_as_longlong(mx[q])));
        }
        sync_round(tag);
    };
    if (p.use_tma) {
      if constexpr (FUSE == 3) {
        // Fused three-term sweeps; decisions term by term as the reference's loop
        // (expact.cpp:81-95) on the six maxima of each sweep.  State between sweeps:
        // (T_j in T[tsel^1], F_{j-1} in F[fsel^1]) with F_j = F_{j-1} + T_j implicit.
        int fsel = 0, tsel = 0;
        for (int stage = 0; stage < s_st; ++stage) {
            const int fstart = stage_start(stage);
            if (fstart == kBufF0) fsel = 1;
            else if (fstart == kBufF1) fsel = 0;
            int used = 0;
            int kind = fstart < 0 ? k2FirstZero : (bordered ? k2FirstBorder : k2FirstPlain);
            int xb = fstart, fb = -1;
            while (true) {
                const double c1 = __ddiv_rn(tau_s, static_cast<double>(used + 1));  // expact.cpp:83
                const double c2 = __ddiv_rn(tau_s, static_cast<double>(used + 2));
                const double c3 = __ddiv_rn(tau_s, static_cast<double>(used + 3));
                const int fout = kBufF0 + fsel, tout = kBufT0 + tsel;
                double mx[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                {
                    const int xb_ = xb < 0 ? 0 : xb, fb_ = fb < 0 ? 0 : fb;
                    double* oT = p.buf[tout];
                    double* oF = p.buf[fout];
                    if (kind == k2Next)
                        sweep3_tma<k2Next>(p, ring3, xb_, fb_, c1, c2, c3, oT, oF, mx, seq3x, seq3f, pm3x, pm3f,
                                           sm.wtab);
                    else if (kind == k2FirstBorder)
                        sweep3_tma<k2FirstBorder>(p, ring3, xb_, fb_, c1, c2, c3, oT, oF, mx, seq3x, seq3f, pm3x,
                                                  pm3f, sm.wtab);
                    else if (kind == k2FirstZero)
                        sweep3_tma<k2FirstZero>(p, ring3, xb_, fb_, c1, c2, c3, oT, oF, mx, seq3x, seq3f, pm3x,
                                                pm3f, sm.wtab);
                    else
                        sweep3_tma<k2FirstPlain>(p, ring3, xb_, fb_, c1, c2, c3, oT, oF, mx, seq3x, seq3f, pm3x,
                                                 pm3f, sm.wtab);
                }
                block_reduce<6, true>(mx, sm);
                publish_max(mx, 6, kind == k2Next ? kTrFusedNext : kTrFusedFirst);
                const unsigned long long* sl = p.slots + ((round - 1) % 3) * 8;
                double cur[3], fn[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    cur[k] = slot_read(sl + 2 * k);
                    fn[k] = slot_read(sl + 2 * k + 1);
                    if (bordered) fn[k] = nan_dropping_max(fn[k], 1.0);  // f_n == 1 (expact.cpp:89)
                }
                // term used+1: F1 = Fprev + T1 was not stored -- recompute it if the stage ends here
                ++used;
                if (!finite_or_fail(cur[0], fn[0])) return;
                if (__dadd_rn(prev, cur[0]) <= __dmul_rn(p.tol, fn[0]) || used == m_deg) {
                    double* Fo = p.buf[fout];
                    if (kind == k2FirstZero) {
                        sweep_points(op, [&](int64_t v) {
                            Fo[v] = __dadd_rn(0.0, __dmul_rn(c1, __dadd_rn(0.0, G[v])));
                        });
                    } else if (kind == k2FirstBorder) {
                        stencil_sweep(p, sm, ring, seq, xb, -1, kBufG, [&](int64_t v, double acc, double x, double,
                                                                           double bg) {
                            Fo[v] = __dadd_rn(x, __dmul_rn(c1, __dadd_rn(acc, bg)));
                        });
                    } else if (kind == k2FirstPlain) {
                        stencil_sweep(p, sm, ring, seq, xb, -1, -1, [&](int64_t v, double acc, double x, double,
                                                                        double) {
                            Fo[v] = __dadd_rn(x, __dmul_rn(c1, acc));
                        });
                    } else {
                        stencil_sweep(p, sm, ring, seq, xb, fb, -1, [&](int64_t v, double acc, double x, double f,
                                                                        double) {
                            Fo[v] = __dadd_rn(__dadd_rn(f, x), __dmul_rn(c1, acc));
                        });
                    }
                    gsync(kTrTerm);
                    prev = fn[0];
                    fres = fout;
                    tres = -1;
                    break;
                }
                prev = cur[0];
                // term used+1: F2, stored
                ++used;
                if (!finite_or_fail(cur[1], fn[1])) return;
                if (__dadd_rn(prev, cur[1]) <= __dmul_rn(p.tol, fn[1]) || used == m_deg) {
                    prev = fn[1];
                    fres = fout;
                    tres = -1;
                    break;
                }
                prev = cur[1];
                // term used+1: F3 = F2 + T3, implicit
                ++used;
                if (!finite_or_fail(cur[2], fn[2])) return;
                if (__dadd_rn(prev, cur[2]) <= __dmul_rn(p.tol, fn[2]) || used == m_deg) {
                    prev = fn[2];
                    fres = fout;
                    tres = tout;
                    break;
                }
                prev = cur[2];
                kind = k2Next;
                xb = tout;
                fb = fout;
                fsel ^= 1;
                tsel ^= 1;
            }
            total_terms += used;
            if (info && stage < kMaxLoggedStages) info->terms[stage] = used;
        }
      } else {
        // Fused two-term sweeps; the decisions are taken term by term exactly as the
        // reference's loop (expact.cpp:81-95), on the four maxima of each sweep.
        //
        // The sweep first computes bounding maxima (max_key: the high words of |x|), and the
        // decisions are taken on intervals: by the monotonicity of rounded + and *, a test is
        // settled when fl(U_prev + U_cur) <= fl(tol * L_f) (the reference stops) or
        // fl(L_prev + L_cur) > fl(tol * U_f) (it goes on), and so is every later use of the
        // bounds.  Otherwise (a test within ~2^-20 of its threshold, or an inf/NaN anywhere)
        // the same sweep runs again with exact NaN-dropping maxima -- its outputs are
        // rewritten with the same bits -- plus the exact max|X| of its input, which is the
        // exact value of an inexact `prev` (prev is ||T_j|| = ||X|| inside a stage and
        // ||f|| = ||X|| (merged with f_n = 1 when bordered) at a stage's first sweep), and the
        // reference's tests run on exact values.  SolveParams::exact_max = 1 always runs the
        // exact sweep, 2 always reruns (test modes).
        //
        // A stage that ended on an implicit F + T starts from it without storing f: its first
        // sweep sums the two in shared memory (sweep2_tma with the Ring2I layout).
        int fsel = 0, tsel = 0;
        double prevU = prev;  // prev's upper bound; prev (the lower bound) == prevU when exact
        for (int stage = 0; stage < s_st; ++stage) {
            const int fstart = stage == 0 ? (bordered ? -1 : kBufG) : fres;
            int timp = stage == 0 ? -1 : tres;  // f = F[fstart] + T[timp] when timp >= 0
            if (fstart == kBufF0) fsel = 1;
            else if (fstart == kBufF1) fsel = 0;
            if (timp == kBufT0) tsel = 1;
            else if (timp == kBufT1) tsel = 0;
            int used = 0;
            int kind = fstart < 0 ? k2FirstZero : (bordered ? k2FirstBorder : k2FirstPlain);
            int xb = fstart, fb = -1;
            while (true) {
                const double c1 = __ddiv_rn(tau_s, static_cast<double>(used + 1));  // expact.cpp:83
                const double c2 = __ddiv_rn(tau_s, static_cast<double>(used + 2));
                const int fout = kBufF0 + fsel, tout = kBufT0 + tsel;
                auto run_sweep = [&](auto exactc, double (&mx)[5]) __attribute__((always_inline)) {
                    constexpr bool kEx = decltype(exactc)::value;
                    const int xb_ = xb < 0 ? 0 : xb, fb_ = fb < 0 ? 0 : fb;
                    double* oT = p.buf[tout];
                    double* oF = p.buf[fout];
                    constexpr bool kSkip = FUSE == 4;
                    if (kind == k2Next)
                        sweep2_tma<k2Next, kSkip, kEx>(p, ring2, xb_, fb_, kBufG, c1, c2, oT, oF, mx, seq2, pmask2,
                                                       sm.wtab);
                    else if (timp >= 0 && kind == k2FirstBorder)
                        sweep2_tma<k2FirstBorder, kSkip, kEx>(p, ring2i, xb_, timp, kBufG, c1, c2, oT, oF, mx, seq2,
                                                              pmask2, sm.wtab);
                    else if (timp >= 0)
                        sweep2_tma<k2FirstPlain, kSkip, kEx>(p, ring2i, xb_, timp, kBufG, c1, c2, oT, oF, mx, seq2,
                                                             pmask2, sm.wtab);
                    else if (kind == k2FirstBorder)
                        sweep2_tma<k2FirstBorder, kSkip, kEx>(p, ring2, xb_, fb_, kBufG, c1, c2, oT, oF, mx, seq2,
                                                              pmask2, sm.wtab);
                    else if (kind == k2FirstZero)
                        sweep2_tma<k2FirstZero, kSkip, kEx>(p, ring2, xb_, fb_, kBufG, c1, c2, oT, oF, mx, seq2,
                                                            pmask2, sm.wtab);
                    else
                        sweep2_tma<k2FirstPlain, kSkip, kEx>(p, ring2, xb_, fb_, kBufG, c1, c2, oT, oF, mx, seq2,
                                                             pmask2, sm.wtab);
                    if (!kEx && p.xchg) {
                        // (every thread's generic -> async-proxy fence: the end of sweep2_tma)
                        xchg_keys4(p, sm, mx, xround++);
                        trace_mark(p, kind == k2Next ? kTrFusedNext : kTrFusedFirst);
                        return;
                    }
                    block_reduce<5, true>(mx, sm);
                    if (threadIdx.x == 0) {
                        unsigned long long* sl = p.slots + (round % 3) * 8;
#pragma unroll
                        for (int q = 0; q < 5; ++q)
                            if (mx[q] > 0.0) atomicMax(sl + q, static_cast<unsigned long long>(__double_as_longlong(mx[q])));
                    }
                    sync_round(kind == k2Next ? kTrFusedNext : kTrFusedFirst);
                    const unsigned long long* sl = p.slots + ((round - 1) % 3) * 8;
#pragma unroll
                    for (int q = 0; q < 5; ++q) mx[q] = slot_read(sl + q);
                };
                // maxima: [0] |T1|, [1] |F1|, [2] |T2|, [3] |F2|, [4] |X| (exact sweep only)
                double lo[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                if (p.exact_max != 1) {
                    run_sweep(std::false_type{}, lo);
                    // settle both tests on the bounds, or fall back to the exact sweep
                    double fL[2] = {lo[1], lo[3]}, fU[2] = {key_upper(lo[1]), key_upper(lo[3])};
                    const double cL[2] = {lo[0], lo[2]}, cU[2] = {key_upper(lo[0]), key_upper(lo[2])};
                    if (bordered)
                        for (int k = 0; k < 2; ++k) {
                            fL[k] = nan_dropping_max(fL[k], 1.0);  // f_n == 1 (expact.cpp:89)
                            fU[k] = nan_dropping_max(fU[k], 1.0);
                        }
                    bool settled = p.exact_max != 2 && !isinf(lo[0]) && !isinf(lo[1]) && !isinf(lo[2]) &&
                                   !isinf(lo[3]);
                    // test of term used+k+1 on bounds: 1 stop, 0 go on, -1 unsettled
                    auto test = [&](int k, double pl, double pu, double cl, double cu, double fl, double fu) {
                        if (used + k + 1 == m_deg || __dadd_rn(pu, cu) <= __dmul_rn(p.tol, fl)) return 1;
                        return __dadd_rn(pl, cl) <= __dmul_rn(p.tol, fu) ? -1 : 0;
                    };
                    int stop = 0;  // 1: after T1, 2: after T2
                    if (settled) {
                        const int a = test(0, prev, prevU, cL[0], cU[0], fL[0], fU[0]);
                        if (a < 0) settled = false;
                        else if (a == 1) stop = 1;
                        else {
                            const int b = test(1, cL[0], cU[0], cL[1], cU[1], fL[1], fU[1]);
                            if (b < 0) settled = false;
                            else if (b == 1) stop = 2;
                        }
                    }
                    if (settled) {
                        if (stop == 1) {
                            ++used;
                            prev = fL[0];
                            prevU = fU[0];
                            fres = fout;
                            tres = -1;
                            break;
                        }
                        used += 2;
                        if (stop == 2) {
                            prev = fL[1];
                            prevU = fU[1];
                            fres = fout;
                            tres = tout;
                            break;
                        }
                        prev = cL[1];
                        prevU = cU[1];
                        kind = k2Next;
                        timp = -1;
                        xb = tout;
                        fb = fout;
                        fsel ^= 1;
                        tsel ^= 1;
                        continue;
                    }
                    for (int q = 0; q < 5; ++q) lo[q] = 0.0;
                    ++reruns;
                }
                run_sweep(std::true_type{}, lo);  // one call site per instantiation: all inlined
                // exact maxima: the reference's tests verbatim
                if (prev != prevU) {  // prev = ||X|| (stage start: ||f|| with f_n = 1 merged)
                    prev = (kind != k2Next && bordered) ? nan_dropping_max(lo[4], 1.0) : lo[4];
                }
                double cur[2] = {lo[0], lo[2]};
                double fn[2] = {lo[1], lo[3]};
                if (bordered) {
                    fn[0] = nan_dropping_max(fn[0], 1.0);  // f_n == 1 (expact.cpp:89)
                    fn[1] = nan_dropping_max(fn[1], 1.0);
                }
                // term used+1 (result F1, explicit)
                ++used;
                if (!finite_or_fail(cur[0], fn[0])) return;
                if (__dadd_rn(prev, cur[0]) <= __dmul_rn(p.tol, fn[0]) || used == m_deg) {
                    prev = prevU = fn[0];
                    fres = fout;
                    tres = -1;
                    break;
                }
                prev = cur[0];
                // term used+1 (result F2 = F1 + T2, implicit)
                ++used;
                if (!finite_or_fail(cur[1], fn[1])) return;
                if (__dadd_rn(prev, cur[1]) <= __dmul_rn(p.tol, fn[1]) || used == m_deg) {
                    prev = prevU = fn[1];
                    fres = fout;
                    tres = tout;
                    break;
                }
                prev = prevU = cur[1];
                kind = k2Next;
                timp = -1;
                xb = tout;
                fb = fout;
                fsel ^= 1;
                tsel ^= 1;
            }
            total_terms += used;
            if (info && stage < kMaxLoggedStages) info->terms[stage] = used;
        }
      }
    } else {
        // Single-term sweeps (shapes the TMA path cannot describe)
        int fcur = bordered ? -1 : kBufG;  // -1: f = e_{n+1} (all zero) for the bordered action
        int tprev = -1;
        int fsel = 0, tsel = 0;
        for (int stage = 0; stage < s_st; ++stage) {
            int used = 0;
            for (int j = 1; j <= m_deg; ++j) {
                const double c = __ddiv_rn(tau_s, static_cast<double>(j));  // expact.cpp:83
                const TermKind kind = j > 1 ? kNext : (fcur < 0 ? kFirstZero : (bordered ? kFirstBorder : kFirstPlain));
                const int fout = kBufF0 + fsel;
                const int tout = kBufT0 + tsel;
                double* Fo = p.buf[fout];
                double* To = p.buf[tout];
                double mt = 0.0, mf = 0.0;
                // term = c * (A~ term); f += term   (expact.cpp:82-87)
                auto emit = [&](int64_t v, double sc, double fin) {
                    const double tn = __dmul_rn(c, sc);
                    const double fnv = __dadd_rn(fin, tn);
                    To[v] = tn;
                    Fo[v] = fnv;
                    mt = nan_dropping_max(mt, fabs(tn));
                    mf = nan_dropping_max(mf, fabs(fnv));
                };
                if (kind == kFirstZero) {
                    // A~ e_{n+1} = the border column b/gamma; f was e_{n+1}
                    sweep_points(op, [&](int64_t v) { emit(v, __dadd_rn(0.0, G[v]), 0.0); });
                } else if (kind == kFirstBorder) {
                    // the border entry (column n, b_i/gamma) is last in its row; term_n = 1 only
                    // on a stage's first term (expact.cpp:137-138, :96)
                    stencil_sweep(p, sm, ring, seq, fcur, -1, kBufG, [&](int64_t v, double acc, double f, double, double bg) {
                        emit(v, __dadd_rn(acc, bg), f);
                    });
                } else if (kind == kFirstPlain) {
                    stencil_sweep(p, sm, ring, seq, fcur, -1, -1,
                                  [&](int64_t v, double acc, double f, double, double) { emit(v, acc, f); });
                } else {
                    stencil_sweep(p, sm, ring, seq, tprev, fcur, -1,
                                  [&](int64_t v, double acc, double, double f, double) { emit(v, acc, f); });
                }
                double v2[2] = {mt, mf};
                block_reduce<2, true>(v2, sm);
                if (threadIdx.x == 0) {
                    unsigned long long* sl = p.slots + (round % 3) * 8;
                    if (v2[0] > 0.0) atomicMax(sl + 0, static_cast<unsigned long long>(__double_as_longlong(v2[0])));
                    if (v2[1] > 0.0) atomicMax(sl + 1, static_cast<unsigned long long>(__double_as_longlong(v2[1])));
                }
                sync_round(kTrTerm);
                ++used;
                fcur = fout;
                tprev = tout;
                fsel ^= 1;
                tsel ^= 1;
                const unsigned long long* sl = p.slots + ((round - 1) % 3) * 8;
                const double cur = slot_read(sl + 0);
                double fnorm = slot_read(sl + 1);
                if (bordered) fnorm = nan_dropping_max(fnorm, 1.0);  // f_n == 1 (expact.cpp:89)
                if (!finite_or_fail(cur, fnorm)) return;
                if (__dadd_rn(prev, cur) <= __dmul_rn(p.tol, fnorm)) {  // expact.cpp:93
                    prev = fnorm;  // next stage: term = f, ||term|| = ||f|| (expact.cpp:80, :96)
                    break;
                }
                prev = (j == m_deg) ? fnorm : cur;
            }
            total_terms += used;
            if (info && stage < kMaxLoggedStages) info->terms[stage] = used;
        }
        fres = fcur;
    }
    if (info) {
        info->total_terms = total_terms;
        info->reruns = reruns;
    }
    if (leader) {
        if (p.xchg) ctrl->xround = xround;
        ctrl->fres = fres;
        ctrl->tres = tres;
        ctrl->last_terms = static_cast<int>(total_terms);
    }
    if (p.use_tma) fence_proxy_async_global();
}

#ifndef GS_TILE8  // (the 2-D kernel's thread mapping needs the default 512 threads)
#include "gs_flat2d.cuh"
#endif

__global__ void advance_kernel(Ctrl* ctrl) { ctrl->step += 1; }

// ------------------------------------------------------------------------------------------
// K5 update: u <- u + tau * (gamma/tau) * y (run, + compute_metrics) or out = scale * y
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ void update_body(const SolveParams& p, int step) {
    if (step < 0) step = __ldcg(&p.ctrl->step);  // graph replay: the step lives on the device
    __shared__ Smem sm;
    const Ctrl* ctrl = p.ctrl;
    // The Taylor kernel leaves its last round's maxima in one rotating slot; the next step's
    // first rounds expect all three slots zero (their atomicMax would otherwise see the stale
    // ||f|| of the previous step's last sweep).  The Taylor kernel has finished: stream order.
    if (vcta() == 0 && threadIdx.x < kSlotWords) p.slots[threadIdx.x] = 0ull;
    if (__ldcg(&ctrl->status)) return;
    trace_mark(p, kTrUpdateIn);
    const int branch = __ldcg(&ctrl->branch);
    const int fres = __ldcg(&ctrl->fres), tres = __ldcg(&ctrl->tres);
    const double t = p.tau;
    const bool bordered = p.mode != kModeExpmv;
    const double* G = p.buf[kBufG];
    const double* F = fres >= 0 ? p.buf[fres] : G;
    const double* TI = tres >= 0 ? p.buf[tres] : nullptr;  // implicit F2 = F1 + T2
    const double* INC = p.buf[kBufT0];
    double* const U = p.buf[kBufU];
    double* const OUT = p.buf[kBufOut];
    // phi1v's result before the step's u + tau * incr (expact.cpp:149-151 / :108-121)
    const double scl = (branch == 0 && bordered) ? __ddiv_rn(__ldcg(&ctrl->gamma), t) : 1.0;
    auto incr = [&](int64_t v) -> double {
        if (branch == 1) return G[v];
        if (branch == 2) return 0.0;
        if (branch == 3) return INC[v];
        const double y = TI ? __dadd_rn(F[v], TI[v]) : F[v];
        return bordered ? __dmul_rn(scl, y) : y;
    };
    if (p.mode == kModeRun) {
        MetricAcc a;
        sweep_points(p.op, [&](int64_t v) {
            const double un = __dadd_rn(U[v], __dmul_rn(t, incr(v)));  // integrator.cpp:59-61
            U[v] = un;
            if (p.want_metrics) a.add(p, v, un);
        });
        if (p.want_metrics) metrics_commit(p, sm, a, step + 1);
        if (p.use_tma) fence_proxy_async_global();
    } else {
        sweep_points(p.op, [&](int64_t v) { OUT[v] = incr(v); });
    }
}

// Software barrier of one CTA group (the ensemble's per-member virtual grid); the pattern of
// cooperative groups' grid.sync: fence, arrive, the last arriver opens the next generation.
struct GroupBarrier {
    unsigned* count;
    unsigned* gen;
    unsigned n;
    __device__ __forceinline__ void sync() const {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned g0 = ld_acquire_gpu(gen);
            __threadfence();
            if (atomicAdd(count, 1u) == n - 1) {
                atomicExch(count, 0u);
                __threadfence();
                atomicAdd(gen, 1u);
            } else {
                while (ld_acquire_gpu(gen) == g0) {
                }
            }
            __threadfence();
        }
        __syncthreads();
    }
};

#ifndef GS_TILE8
__global__ void __launch_bounds__(kSolveThreads) taylor2d_kernel(const __grid_constant__ SolveParams p, int border_blocks,
                                                                  int step) {
    vgrid_set(blockIdx.x, gridDim.x);
    cg::grid_group grid = cg::this_grid();
    taylor2d_body(p, border_blocks, step, [&] { grid.sync(); });
}
#endif

template <int FUSE>
__global__ void __launch_bounds__(kSolveThreads, kMinBlocks) taylor_kernel(const __grid_constant__ SolveParams p,
                                                                  int border_blocks, int step) {
    vgrid_set(blockIdx.x, gridDim.x);
    cg::grid_group grid = cg::this_grid();
    taylor_body<FUSE>(p, border_blocks, step, [&] { grid.sync(); }, false);
}

// Ensemble Taylor kernel (cooperative): the grid is cut into gridDim.x / group CTA groups; each
// group takes members from a queue and runs a member's whole Taylor loop on its virtual grid,
// with a software group barrier in place of grid.sync.  ctl: per group {count, gen, member[2]}
// followed by the queue head, zeroed before the launch.
// The first `extra` groups have group + 1 CTAs (so the launch can fill every SM); a member's
// TMA work split (cta_work) follows the group's actual CTA count.
template <int FUSE>
__global__ void __launch_bounds__(kSolveThreads, kMinBlocks) ens_taylor_kernel(const SolveParams* __restrict__ P, int n_members,
                                                                      int group, int border_blocks, int step,
                                                                      unsigned* ctl, const unsigned* order, int extra) {
    const int big = group + 1;
    int g, size, r;
    if (static_cast<int>(blockIdx.x) < extra * big) {
        g = blockIdx.x / big;
        r = blockIdx.x % big;
        size = big;
    } else {
        const int b = blockIdx.x - extra * big;
        g = extra + b / group;
        r = b % group;
        size = group;
    }
    vgrid_set(r, size);
    const int ngroups = extra + (gridDim.x - extra * big) / group;
    unsigned* mine = ctl + 4 * g;
    unsigned* queue = ctl + 4 * ngroups;
    const GroupBarrier bar{mine, mine + 1, static_cast<unsigned>(size)};
    bool reinit = false;
    for (int it = 0;; ++it) {
        // the group leader takes the next member; slots alternate so that a CTA still reading
        // this iteration's never sees the next one's (the leader passes a group barrier first)
        if (vcta() == 0 && threadIdx.x == 0) mine[2 + (it & 1)] = atomicAdd(queue, 1u);
        bar.sync();
        const int q = static_cast<int>(__ldcg(mine + 2 + (it & 1)));
        if (q >= n_members) return;  // uniform within the group
        const int m = static_cast<int>(__ldg(order + q));
        taylor_body<FUSE>(P[m], border_blocks, step, [&] { bar.sync(); }, reinit);
        reinit = true;
    }
}

// ------------------------------------------------------------------------------------------
// Kernels of one member (plain launches) and their ensemble forms: CTA b of an ensemble launch
// works for member b / cpm as CTA b % cpm of cpm.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kSolveThreads) metrics_kernel(const __grid_constant__ SolveParams p) {
    vgrid_set(blockIdx.x, gridDim.x);
    metrics_body(p);
}
__global__ void __launch_bounds__(kSolveThreads, kMinBlocks) prep_kernel(const __grid_constant__ SolveParams p, int step) {
    vgrid_set(blockIdx.x, gridDim.x);
    prep_body(p, step);
}
__global__ void __launch_bounds__(kSolveThreads) border_kernel(const __grid_constant__ SolveParams p, int prep_blocks,
                                                               int step) {
    vgrid_set(blockIdx.x, gridDim.x);
    border_body(p, prep_blocks, step);
}
__global__ void __launch_bounds__(kSolveThreads, 2) seqsum_tiles_kernel(const __grid_constant__ SolveParams p, int which) {
    vgrid_set(blockIdx.x, gridDim.x);
    seqsum_tiles_body(p, which);
}
__global__ void __launch_bounds__(kSolveThreads) seqsum_items_kernel(const __grid_constant__ SolveParams p, int which) {
    vgrid_set(blockIdx.x, gridDim.x);
    seqsum_items_body(p, which);
}
__global__ void __launch_bounds__(kSolveThreads, 2) ens_seqsum_tiles_kernel(const SolveParams* __restrict__ P, int cpm,
                                                                         int which) {
    vgrid_set(blockIdx.x % cpm, cpm);
    seqsum_tiles_body(P[blockIdx.x / cpm], which);
}
__global__ void __launch_bounds__(kSolveThreads) ens_seqsum_items_kernel(const SolveParams* __restrict__ P, int cpm,
                                                                         int which) {
    vgrid_set(blockIdx.x % cpm, cpm);
    seqsum_items_body(P[blockIdx.x / cpm], which);
}
__global__ void __launch_bounds__(kSolveThreads) update_kernel(const __grid_constant__ SolveParams p, int step) {
    vgrid_set(blockIdx.x, gridDim.x);
    update_body(p, step);
}
__global__ void __launch_bounds__(kSolveThreads) ens_metrics_kernel(const SolveParams* __restrict__ P, int cpm) {
    vgrid_set(blockIdx.x % cpm, cpm);
    metrics_body(P[blockIdx.x / cpm]);
}
__global__ void __launch_bounds__(kSolveThreads, kMinBlocks) ens_prep_kernel(const SolveParams* __restrict__ P, int cpm, int step) {
    vgrid_set(blockIdx.x % cpm, cpm);
    prep_body(P[blockIdx.x / cpm], step);
}
__global__ void __launch_bounds__(kSolveThreads) ens_border_kernel(const SolveParams* __restrict__ P, int cpm,
                                                                   int prep_blocks, int step) {
    vgrid_set(blockIdx.x % cpm, cpm);
    border_body(P[blockIdx.x / cpm], prep_blocks, step);
}
__global__ void __launch_bounds__(kSolveThreads) ens_update_kernel(const SolveParams* __restrict__ P, int cpm, int step) {
    vgrid_set(blockIdx.x % cpm, cpm);
    update_body(P[blockIdx.x / cpm], step);
}

template __global__ void taylor_kernel<2>(const __grid_constant__ SolveParams, int, int);
#ifndef GS_TILE8
template __global__ void taylor_kernel<3>(const __grid_constant__ SolveParams, int, int);
#endif
template __global__ void taylor_kernel<4>(const __grid_constant__ SolveParams, int, int);
template __global__ void ens_taylor_kernel<2>(const SolveParams*, int, int, int, int, unsigned*, const unsigned*, int);
template __global__ void ens_taylor_kernel<4>(const SolveParams*, int, int, int, int, unsigned*, const unsigned*, int);

// The queue's order for the next Taylor launch: members by their last step's Taylor terms,
// most first (ties by index) -- the longest runs start first, so the groups finish together
// (longest-processing-time-first).  Before the first step every count is 0: index order.
__global__ void ens_order_kernel(const SolveParams* __restrict__ P, int n_members, unsigned* order) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_members; i += gridDim.x * blockDim.x) {
        const int wi = __ldcg(&P[i].ctrl->last_terms);
        int rank = 0;
        for (int j = 0; j < n_members; ++j) {
            const int wj = __ldcg(&P[j].ctrl->last_terms);
            rank += (wj > wi) || (wj == wi && j < i);
        }
        order[rank] = static_cast<unsigned>(i);
    }
}


// Host-side handles of the instantiations (kept in this translation unit).
const void* taylor_kernel_fn(int fuse) {
#ifdef GS_TILE8
    // the three-term rings need more threads than a 64 x 8 tile has
    return fuse == 4 ? reinterpret_cast<const void*>(taylor_kernel<4>) : reinterpret_cast<const void*>(taylor_kernel<2>);
#else
    return fuse == 3   ? reinterpret_cast<const void*>(taylor_kernel<3>)
           : fuse == 4 ? reinterpret_cast<const void*>(taylor_kernel<4>)
                       : reinterpret_cast<const void*>(taylor_kernel<2>);
#endif
}
const void* taylor2d_kernel_fn() {
#ifndef GS_TILE8
    return reinterpret_cast<const void*>(taylor2d_kernel);
#else
    return nullptr;
#endif
}
const void* ens_taylor_kernel_fn(int fuse) {
    return fuse == 4 ? reinterpret_cast<const void*>(ens_taylor_kernel<4>)
                     : reinterpret_cast<const void*>(ens_taylor_kernel<2>);
}

}  // namespace gs
