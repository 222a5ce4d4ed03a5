// gs_cluster.cu -- small grids: whole exponential-Euler runs inside one thread-block cluster.
//
// For grids whose state fits in the distributed shared memory of one 16-CTA cluster (up to
// 40 K voxels: C1 32^3; C2 256^2 does not fit beside the exact-sum item lists and takes the
// 2-D resident-tile kernel, gs_flat2d.cuh), the launch sequence of the large-grid path (prep,
// border, cooperative Taylor, update, each with grid-wide barriers) is replaced by ONE
// persistent launch that runs every step of gs_run:
//   * the voxels are split into 16 contiguous slices, one per CTA; every vector of the step
//     (u, b/gamma, f x2, term x2) lives in shared memory, with a halo of one plane (one
//     row in 2-D) on each side that is pulled from the neighbour CTAs over DSMEM after the
//     producing pass;
//   * reductions (||b||_1, the bordered column sum, the per-term maxima, the metrics) go
//     through a per-CTA mailbox read by every CTA over DSMEM in rank order, so each CTA
//     takes the same decisions from the same values (sums in a fixed order, maxima order-free);
//   * barrier.cluster replaces the grid barrier (one per Taylor term).
// The arithmetic is the large-grid path's operation for operation (row_apply in CSR column
// order, the same termination tests, expact.cpp:63-153; integrator.cpp:52-89).
#include <cooperative_groups.h>
#include <cstdio>

#include "gs_kernels.cuh"

namespace cg = cooperative_groups;

namespace gs {

namespace {

#include "gs_seqsum.cuh"

constexpr int kCT = kSolveThreads;  // threads per CTA

struct ClusterShared {
    double wtab[256];
    double red[kCT / 32][4];
    double mbox[2][4];  // per-CTA results of the last reduction, double-buffered by parity
    double bcast[4];    // the cluster-combined values, broadcast inside the CTA
};

// Neighbour-presence bits of a voxel (x-, x+, y-, y+, z-, z+), precomputed once per launch.
enum : uint8_t { kHx0 = 1, kHx1 = 2, kHy0 = 4, kHy1 = 8, kHz0 = 16, kHz1 = 32 };

// Warp 0 combines the ranks' mailboxes into cs.bcast[0..K): lane r loads rank r's entries
// (one DSMEM round trip instead of K x ranks serial ones); sums are added in rank order,
// maxima (kind 1: non-negative, start 0; kind 2: signed, start -inf) reduced order-free.
// Every thread must call it (it ends with a block barrier).
template <int K>
__device__ __forceinline__ void cl_combine(cg::cluster_group& cl, ClusterShared& cs, int par, const int (&kind)[K]) {
    const int nr = static_cast<int>(cl.num_blocks());
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double v[K];
        const double* mb = lane < nr ? cl.map_shared_rank(&cs.mbox[par][0], lane) : nullptr;
#pragma unroll
        for (int q = 0; q < K; ++q) v[q] = mb ? mb[q] : (kind[q] == 2 ? -INFINITY : 0.0);
#pragma unroll
        for (int q = 0; q < K; ++q) {
            if (kind[q] == 0) {
                double acc = __shfl_sync(0xffffffffu, v[q], 0);
                for (int r = 1; r < nr; ++r) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, v[q], r));
                if (lane == 0) cs.bcast[q] = acc;
            } else {
                const double m = warp_max(v[q]);
                if (lane == 0) cs.bcast[q] = m;
            }
        }
    }
    __syncthreads();
}

// select_params (expact.cpp:29-61) with r_m from the host's libm: as in gs_solve.cu
__device__ int cluster_select_params(double norm_tA, const double* rtab, int* s_out, int* m_out) {
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

// Block reduction into mbox[par][0..K): sums (fixed tree) or maxima per entry kind.
template <int K>
__device__ __forceinline__ void block_to_mbox(ClusterShared& cs, int par, double (&v)[K], const bool (&is_max)[K]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = is_max[q] ? warp_max(v[q]) : warp_sum(v[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < K; ++q) cs.red[wid][q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            double a = cs.red[0][q];
            for (int w = 1; w < kCT / 32; ++w)
                a = is_max[q] ? nan_dropping_max(a, cs.red[w][q]) : __dadd_rn(a, cs.red[w][q]);
            cs.mbox[par][q] = a;
        }
    }
}

// The reference's sequential sum of |B| over the cluster's slices in rank order (= index
// order), exactly (gs_seqsum.cuh): each CTA builds the run / raw items of its slice from an
// approximate prefix (the ranks' tree partials in mbox[par][0], after a cluster barrier);
// after a second barrier every CTA gathers all ranks' lists over DSMEM and walks them the same
// way, so all CTAs hold the same value.  A list longer than kClItemCap is walked element by
// element over DSMEM, followed by one more barrier (uniform: every CTA sees the same counts)
// before anyone overwrites B.
constexpr int kClEPT = 8;  // elements per thread: slices of up to kCT * 8 voxels
struct ClusterSeq {        // static shared memory
    SeqSmem sm;
    seq::Item own[kClItemCap];
    int count, pref[kClusterCTAs + 1];
    int walked;  // this CTA's walk read remote B (a fallback)
    unsigned flags;
    double result, prefix;
};
// The gathered sequence, staged for seq_walk_batch, in dynamic shared memory over F0..T1
// (cluster_b_offset keeps kClGatherDoubles there).
struct ClusterGather {
    int* kind;
    int* B;
    uint64_t *d0, *d1, *lo, *hi;
    longlong2* pos;
    __device__ explicit ClusterGather(void* base) {
        unsigned char* b = static_cast<unsigned char*>(base);
        pos = reinterpret_cast<longlong2*>(b);
        d0 = reinterpret_cast<uint64_t*>(b + 16 * kClAll);
        d1 = d0 + kClAll;
        lo = d1 + kClAll;
        hi = lo + kClAll;
        kind = reinterpret_cast<int*>(hi + kClAll);
        B = kind + kClAll;
    }
};
static_assert(56 * kClAll <= 8 * kClGatherDoubles, "gather layout");

__device__ double cl_exact_sum(cg::cluster_group& cl, ClusterShared& cs, ClusterSeq& q, void* gather, int par,
                               const double* B, int64_t len, int64_t lo, int64_t S, int64_t N, int rank, int nranks,
                               bool debug) {
    const int tid = threadIdx.x;
    // 16-byte aligned (its start/len pairs are 16-byte loads); F0 may start 8 bytes off
    const ClusterGather g(reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(gather) + 15) & ~uintptr_t(15)));
    // approximate sum before this slice; this slice's non-finite flags
    if (tid < 32) {
        double v = tid < rank ? *cl.map_shared_rank(&cs.mbox[par][0], tid) : 0.0;
        v = warp_sum(v);
        if (tid == 0) {
            q.prefix = v;
            q.flags = 0u;
            seq_open_reset(q.sm);
        }
    }
    double xv[kClEPT];
    unsigned f = 0;
#pragma unroll
    for (int j = 0; j < kClEPT; ++j) {
        const int64_t e = static_cast<int64_t>(tid) * kClEPT + j;
        xv[j] = e < len ? B[e] : 0.0;
        f |= isnan(xv[j]) ? seq::kHasNaN : (isinf(xv[j]) ? seq::kHasInf : 0u);
    }
    __syncthreads();
    f = __reduce_or_sync(0xffffffffu, f);
    if ((tid & 31) == 0 && f) atomicOr(&q.flags, f);
    seq_tile_items<kClEPT>(q.sm, xv, lo, static_cast<int>(len), q.prefix, q.own, kClItemCap);
    if (tid == 0) q.count = len > 0 ? seq_close(q.sm, lo + len, q.own, kClItemCap) : 0;
    cl.sync();
    // every rank's list, compacted in rank order (an overflowed list: one pseudo-item, its range)
    if (tid < 32) {
        int cnt = 0;
        if (tid < nranks) {
            cnt = *cl.map_shared_rank(&q.count, tid);
            cnt = cnt > kClItemCap ? 1 : cnt;
            const unsigned rf = *cl.map_shared_rank(&q.flags, tid);
            if (rf && tid != rank) atomicOr(&q.flags, rf);
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (tid >= o) inc += y;
        }
        if (tid < nranks) q.pref[tid + 1] = inc;
        if (tid == 0) q.pref[0] = 0;
    }
    __syncthreads();
    {
        const int r = tid / kClItemCap, k = tid % kClItemCap;
        if (r < nranks && k < q.pref[r + 1] - q.pref[r]) {
            const int cnt = *cl.map_shared_rank(&q.count, r);
            const int at = q.pref[r] + k;
            seq::Item it;
            if (cnt > kClItemCap) {
                const int64_t rlo = r * S;
                it = seq::Item{seq::kMixed, 0, 0, 0, rlo, min(N, rlo + S) - rlo};
            } else {
                it = cl.map_shared_rank(q.own, r)[k];
            }
            g.kind[at] = it.kind;
            g.B[at] = it.B;
            seq_stage(it.kind, it.B, it.d0, it.d1, g.d0[at], g.d1[at], g.lo[at], g.hi[at]);
            g.pos[at] = make_longlong2(it.start, it.len);
        }
        const int total = q.pref[nranks];
        if (tid < 8) {  // padding of the walk's last batch: zero runs
            g.kind[total + tid] = seq::kEmpty;
            g.B[total + tid] = 0;
            g.d0[total + tid] = g.d1[total + tid] = g.lo[total + tid] = 0ull;
            g.hi[total + tid] = ~0ull;
        }
    }
    __syncthreads();
    bool walked = false;  // a fallback read remote B
    if (tid == 0) {
        uint64_t bits = 0ull;
        bool fin = true;
        if (q.flags & seq::kHasNaN) {
            bits = 0x7ff8000000000000ull;
        } else if (q.flags & seq::kHasInf) {
            bits = 0x7ff0000000000000ull;
        } else {
            fin = seq_walk_batch(bits, g.kind, g.B, g.d0, g.d1, g.lo, g.hi, g.pos, q.pref[nranks],
                                 [&](double a, int64_t l, int64_t h) {
                                     walked = true;
                                     for (int64_t i = l; i < h; ++i) {
                                         const int r = static_cast<int>(i / S);
                                         a = __dadd_rn(a, fabs(cl.map_shared_rank(B, r)[i - r * S]));
                                     }
                                     return a;
                                 },
                                 debug);
            if (!fin) bits = 0x7ff0000000000000ull;
        }
        q.result = __longlong_as_double(static_cast<long long>(bits));
        q.walked = walked ? 1 : 0;
    }
    __syncthreads();
    // a fallback walk read remote B: nobody may overwrite it before everyone is done (uniform:
    // every rank walks the same items with the same state)
    if (q.walked) cl.sync();
    return q.result;
}

}  // namespace

__global__ void __launch_bounds__(kCT, 1) cluster_run_kernel(const __grid_constant__ ClusterParams p) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClusterShared cs;
    __shared__ ClusterSeq csq;
    extern __shared__ __align__(128) unsigned char dyn[];
    const StencilOp& op = p.op;
    const int rank = static_cast<int>(cl.block_rank());
    const int nranks = static_cast<int>(cl.num_blocks());
    const int tid = threadIdx.x;
    const int64_t N = op.n, S = p.slice, H = p.halo;
    const int64_t lo = rank * S, hi = min(N, lo + S);
    const int64_t len = hi > lo ? hi - lo : 0;
    const int64_t HS = S + 2 * H;  // haloed vector length
    // shared layout: U, F0, F1, T0, T1 haloed, then B, then labels
    double* HV[5];
    for (int k = 0; k < 5; ++k) HV[k] = reinterpret_cast<double*>(dyn) + k * HS;
    double* const B = reinterpret_cast<double*>(dyn) + cluster_b_offset(S, H);
    uint8_t* const L = reinterpret_cast<uint8_t*>(B + S);
    uint8_t* const M = L + (S + 15) / 16 * 16;
    enum { kU = 0, kF0 = 1, kF1 = 2, kT0 = 3, kT1 = 4 };
    for (int q = tid; q < 256; q += kCT) cs.wtab[q] = op.wtab[q];
    for (int64_t i = tid; i < len; i += kCT) {
        HV[kU][H + i] = p.u[lo + i];
        L[i] = op.pal[lo + i];
        const int64_t v = lo + i;
        const int x = static_cast<int>(v % op.nx), y = static_cast<int>((v / op.nx) % op.ny),
                  z = static_cast<int>(v / op.sz);
        M[i] = static_cast<uint8_t>((x > 0 ? kHx0 : 0) | (x < op.nx - 1 ? kHx1 : 0) | (y > 0 ? kHy0 : 0) |
                                    (y < op.ny - 1 ? kHy1 : 0) | (z > 0 ? kHz0 : 0) | (z < op.nz - 1 ? kHz1 : 0));
    }
    const bool leader = rank == 0 && tid == 0;
    Ctrl* ctrl = p.ctrl;
    int par = 0;
    cl.sync();

    // neighbours' slices -> this CTA's halo of haloed vector k (after the producing pass)
    auto pull_halo = [&](int k) {
        double* X = HV[k];
        if (rank > 0) {
            const double* R = cl.map_shared_rank(HV[k], rank - 1);
            for (int64_t i = tid; i < H; i += kCT) X[i] = R[H + S - H + i];  // global lo-H+i
        }
        if (rank + 1 < nranks && hi < N) {
            const double* R = cl.map_shared_rank(HV[k], rank + 1);
            const int64_t nh = min(H, N - hi);
            for (int64_t i = tid; i < nh; i += kCT) X[H + S + i] = R[H + i];  // global hi+i
        }
        __syncthreads();
    };
    // y_v = (A x)_v for an own voxel (local index i), x in haloed vector X
    const int sy = static_cast<int>(op.sy), sz = static_cast<int>(op.sz);
    auto apply_row = [&](const double* X, int i) -> double {
        const int li = static_cast<int>(H) + i;
        const unsigned m = M[i];
        RowCoef rc;
        rc.w = cs.wtab[L[i]];
        rc.live = rc.w != 0.0;
        return row_apply(rc, __popc(m), (m & kHz0) ? X[li - sz] : 0.0, (m & kHy0) ? X[li - sy] : 0.0,
                         (m & kHx0) ? X[li - 1] : 0.0, X[li], (m & kHx1) ? X[li + 1] : 0.0,
                         (m & kHy1) ? X[li + sy] : 0.0, (m & kHz1) ? X[li + sz] : 0.0);
    };
    // compute_metrics (integrator.cpp:65-89) of U into metrics[node]
    auto metrics = [&](int node) {
        double v4[4] = {0.0, -INFINITY, -INFINITY, 0.0};  // sum, max, -min, r2
        double mn = INFINITY;
        for (int64_t i = tid; i < len; i += kCT) {
            const double u = HV[kU][H + i];
            v4[0] = __dadd_rn(v4[0], u);
            v4[1] = nan_dropping_max(v4[1], u);
            mn = (u < mn) ? u : mn;
            if (u >= p.front_threshold) {
                const int64_t v = lo + i;
                const int ix = static_cast<int>(v % op.nx);
                const int iy = static_cast<int>((v / op.nx) % op.ny);
                const int iz = static_cast<int>(v / op.sz);
                const double dx = __dsub_rn(__dadd_rn(p.origin[0], __dmul_rn(static_cast<double>(ix), p.h)), p.center[0]);
                const double dy = __dsub_rn(__dadd_rn(p.origin[1], __dmul_rn(static_cast<double>(iy), p.h)), p.center[1]);
                const double dz = __dsub_rn(__dadd_rn(p.origin[2], __dmul_rn(static_cast<double>(iz), p.h)), p.center[2]);
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                v4[3] = nan_dropping_max(v4[3], d2);
            }
        }
        v4[2] = -mn;  // min as a max of the negation (exact)
        const bool km[4] = {false, true, true, true};
        block_to_mbox<4>(cs, par, v4, km);
        cl.sync();
        const int kinds[4] = {0, 2, 2, 1};
        cl_combine<4>(cl, cs, par, kinds);
        if (leader) {
            const double cell = __dmul_rn(__dmul_rn(p.h, p.h), p.h);
            double* out = p.metrics + 4 * node;
            out[0] = __dmul_rn(cell, cs.bcast[0]);
            out[1] = cs.bcast[1];
            out[2] = -cs.bcast[2];
            out[3] = sqrt(cs.bcast[3]);
        }
        par ^= 1;
    };
    if (p.want_metrics) metrics(0);
    pull_halo(kU);

    for (int step = 0; step < p.n_steps; ++step) {
        gs_step_info* info = (p.infos && leader) ? p.infos + step : nullptr;
        const double t = p.tau;
        // ---- RHS g = A u + rho u (1-u) and ||g||_1 (integrator.cpp:54-57, expact.cpp:110)
        double part[1] = {0.0};
        for (int64_t i = tid; i < len; i += kCT) {
            const double u = HV[kU][H + i];
            const double g = __dadd_rn(apply_row(HV[kU], i), __dmul_rn(__dmul_rn(p.rho, u), __dsub_rn(1.0, u)));
            B[i] = g;
            part[0] = __dadd_rn(part[0], fabs(g));
        }
        const bool ks[1] = {false};
        block_to_mbox<1>(cs, par, part, ks);
        cl.sync();
        const int ksum[1] = {0};
        double bnorm;  // expact.cpp:110: the reference's sequential sum (or a rank-order tree sum, A/B)
        if (p.seq_exact) {
            const long long tc = clock64();
            bnorm = cl_exact_sum(cl, cs, csq, HV[kF0], par, B, len, lo, S, N, rank, nranks, p.seq_exact > 1);
            if (p.seq_exact > 1 && leader)
                printf("cluster step %d: bnorm exact sum %lld cycles, %d items\n", step, clock64() - tc,
                       csq.pref[nranks]);
        } else {
            cl_combine<1>(cl, cs, par, ksum);
            bnorm = cs.bcast[0];
        }
        par ^= 1;
        int branch = 0;
        if (t == 0.0) branch = 1;                                  // expact.cpp:108
        else if (bnorm == 0.0) branch = 2;                         // expact.cpp:111
        else if (__dmul_rn(fabs(t), p.anorm) <= 1e-8) branch = 3;  // expact.cpp:114
        const double gamma = branch == 0 ? __ddiv_rn(bnorm, p.anorm) : 0.0;
        if (info) {
            info->s = info->m = 1;
            info->branch = branch;
            info->total_terms = 0;
            info->anorm = p.anorm;
            info->bnorm = bnorm;
            info->gamma = gamma;
            info->coln = info->norm_tA = 0.0;
        }
        int fres = -1;  // haloed vector holding y (the bordered action's f), or -1 for B-based branches
        if (branch == 3) {
            // incr = b + 0.5 t (A b)  (expact.cpp:117-121): B into T0 with its halo
            for (int64_t i = tid; i < len; i += kCT) HV[kT0][H + i] = B[i];
            cl.sync();
            pull_halo(kT0);
            const double ht = __dmul_rn(0.5, t);
            for (int64_t i = tid; i < len; i += kCT)
                HV[kT1][H + i] = __dadd_rn(B[i], __dmul_rn(ht, apply_row(HV[kT0], i)));
            fres = kT1;
        } else if (branch == 0) {
            // b/gamma where b != 0 (expact.cpp:137-138) and the bordered column sum (sparse.cpp:36-38)
            double cs1[1] = {0.0};
            for (int64_t i = tid; i < len; i += kCT) {
                const double b = B[i];
                const double r = (b != 0.0) ? __ddiv_rn(b, gamma) : 0.0;
                B[i] = r;
                cs1[0] = __dadd_rn(cs1[0], fabs(r));
            }
            block_to_mbox<1>(cs, par, cs1, ks);
            cl.sync();
            // sparse.cpp:36-38 on the bordered operator: the sequential sum when the step log asks
            // for it or the rank-order tree sum does not settle (s, m) (seq::coln_settles), else
            // the tree sum, which then selects the same (s, m)
            cl_combine<1>(cl, cs, par, ksum);
            double coln = cs.bcast[0];
            if (p.seq_exact && (p.infos || !seq::coln_settles(t, p.anorm, coln, N, p.rtab, kMaxDegree))) {
                if (p.seq_exact > 1 && leader) printf("cluster step %d: coln exact\n", step);
                coln = cl_exact_sum(cl, cs, csq, HV[kF0], par, B, len, lo, S, N, rank, nranks, p.seq_exact > 1);
            }
            par ^= 1;
            const double norm_tA = __dmul_rn(fabs(t), nan_dropping_max(p.anorm, coln));
            int s_st = 1, m_deg = 1;
            const int sel = cluster_select_params(norm_tA, p.rtab, &s_st, &m_deg);
            if (info) {
                info->coln = coln;
                info->norm_tA = norm_tA;
                info->s = s_st;
                info->m = m_deg;
            }
            if (sel != GS_OK) {
                if (leader) {
                    ctrl->status = sel;
                    ctrl->detail = 1;
                }
                cl.sync();  // uniform branch: no CTA exits while another still reads its mailbox
                return;
            }
            // ---- Taylor stages of single-term passes (expact.cpp:63-99) on [A b/gamma; 0 0]
            const double tau_s = __ddiv_rn(t, static_cast<double>(s_st));
            double prev = 1.0;  // ||e_{n+1}||_inf
            int fcur = -1;      // -1: f = e_{n+1}, all zero in the first n components
            int tprev = -1, fsel = 0, tsel = 0;
            int64_t total_terms = 0;
            for (int stage = 0; stage < s_st; ++stage) {
                int used = 0;
                for (int j = 1; j <= m_deg; ++j) {
                    const double c = __ddiv_rn(tau_s, static_cast<double>(j));  // expact.cpp:83
                    const int fout = kF0 + fsel, tout = kT0 + tsel;
                    double* Fo = HV[fout] + H;
                    double* To = HV[tout] + H;
                    double mm[2] = {0.0, 0.0};
                    for (int64_t i = tid; i < len; i += kCT) {
                        double sc, fin;
                        if (j == 1 && fcur < 0) {  // A~ e_{n+1} = b/gamma; f = e_{n+1}
                            sc = __dadd_rn(0.0, B[i]);
                            fin = 0.0;
                        } else if (j == 1) {       // border entry last in its row, term_n = 1 (expact.cpp:96)
                            sc = __dadd_rn(apply_row(HV[fcur], i), B[i]);
                            fin = HV[fcur][H + i];
                        } else {
                            sc = apply_row(HV[tprev], i);
                            fin = HV[fcur][H + i];
                        }
                        const double tn = __dmul_rn(c, sc);
                        const double fnv = __dadd_rn(fin, tn);
                        To[i] = tn;
                        Fo[i] = fnv;
                        mm[0] = nan_dropping_max(mm[0], fabs(tn));
                        mm[1] = nan_dropping_max(mm[1], fabs(fnv));
                    }
                    const bool kmx[2] = {true, true};
                    block_to_mbox<2>(cs, par, mm, kmx);
                    cl.sync();
                    const int kmax2[2] = {1, 1};
                    cl_combine<2>(cl, cs, par, kmax2);
                    const double cur = cs.bcast[0];
                    const double fnorm = nan_dropping_max(cs.bcast[1], 1.0);  // f_n == 1 (expact.cpp:89)
                    par ^= 1;
                    ++used;
                    fcur = fout;
                    tprev = tout;
                    fsel ^= 1;
                    tsel ^= 1;
                    if (!isfinite(cur) || !isfinite(fnorm)) {  // expact.cpp:90-91
                        if (leader) {
                            ctrl->status = GS_ENUMERIC;
                            ctrl->detail = 2;
                        }
                        cl.sync();  // uniform branch: no CTA exits while another still reads its mailbox
                        return;
                    }
                    if (__dadd_rn(prev, cur) <= __dmul_rn(p.tol, fnorm)) {  // expact.cpp:93
                        prev = fnorm;
                        break;
                    }
                    prev = (j == m_deg) ? fnorm : cur;
                    pull_halo(tout);  // the next term's stencil input
                }
                total_terms += used;
                if (info && stage < kMaxLoggedStages) info->terms[stage] = used;
                if (stage + 1 < s_st) pull_halo(fcur);  // the next stage starts from f
            }
            if (info) info->total_terms = total_terms;
            fres = fcur;
        }
        // ---- u <- u + tau * incr (integrator.cpp:58-61); incr = (gamma/t) y on the Taylor branch
        const double scl = branch == 0 ? __ddiv_rn(gamma, t) : 1.0;
        for (int64_t i = tid; i < len; i += kCT) {
            double incr;
            if (branch == 1) incr = B[i];
            else if (branch == 2) incr = 0.0;
            else if (branch == 3) incr = HV[fres][H + i];
            else incr = __dmul_rn(scl, HV[fres][H + i]);
            HV[kU][H + i] = __dadd_rn(HV[kU][H + i], __dmul_rn(t, incr));
        }
        __syncthreads();
        if (p.want_metrics) metrics(step + 1);
        else cl.sync();
        pull_halo(kU);
    }
    for (int64_t i = tid; i < len; i += kCT) p.u[lo + i] = HV[kU][H + i];
    cl.sync();  // no CTA may exit while others still read its shared memory
}

}  // namespace gs
