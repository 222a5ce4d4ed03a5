// gs_flat2d.cuh -- the Taylor loop of a 2-D grid (nz == 1) with the tile resident in shared memory.
// Included by gs_solve.cu inside its anonymous namespace (it uses that file's block helpers).
//
// expact.cpp:63-99 (expmv) and :101-153 (the bordered action of phi1v) on grids like C2
// (256 x 256 x 1): one CTA per 32 x 32 tile, every CTA resident (cooperative launch).  The TMA
// z-march has nothing to stream here -- one plane -- and pays its pipeline set-up, a grid
// barrier and a maxima round trip for every two terms (6.9 us per sweep measured).  A 2-D tile
// has no z-halo, so deeper temporal blocking is cheap: one ROUND applies K = 4 Taylor terms
// for one barrier.
//   * The CTA keeps X (the current term T_j, or f at a stage start) on its tile plus a K-voxel
//     halo and w, -cnt and b/gamma of the same box in shared memory; each thread owns two tile
//     points, whose f, current term, w and -cnt stay in registers.
//   * Level k = 1..K computes T_k = c_k (A~ T_{k-1}) on the tile grown by K - k voxels (the
//     rim is 21% more points at K = 4, one per thread at most) and, on the tile, f += T_k and
//     the exact NaN-dropping maxima |T_k|, |f| -- the reference's operations in the
//     reference's order (row_apply_nc, the row of the TMA sweeps with its two z-neighbours
//     passed as 0.0), so every value is bitwise the oracle's.
//   * The tile's f after each level and T_K go to global scratch (x2d, two alternating sets).
//     After the barrier the tests of expact.cpp:88-95 run verbatim, term by term, on the 2K
//     grid maxima (the rotating atomicMax slots of the single-term path); they pick the next
//     X -- T_K, or f after the term the stage stopped at -- and each CTA reloads its box from
//     that array (L2).  Terms computed past a stop are discarded, as the reference never
//     computes them.
// The result f is written to F0 (ctrl->fres = F0, explicit).
#pragma once

__shared__ unsigned long long s_max2d[2 * k2dK];  // block maxima of a round
#ifdef GS_2D_PROF
__shared__ long long s_prof[10];
#define PROF(k)                           \
    if (threadIdx.x == 0) {               \
        const long long now_ = clock64(); \
        s_prof[k] += now_ - s_prof[9];    \
        s_prof[9] = now_;                 \
    }
#else
#define PROF(k)
#endif

constexpr int k2dT = 32;               // tile edge
constexpr int k2dP = k2dT + 2 * k2dK;  // box edge and pitch (doubles): tile + halo K
constexpr int k2dBox = k2dP * k2dP;
static_assert(k2dK >= 2 && 2 * k2dK <= kSlots2d, "2K maxima must fit the slots of a round");
static_assert(k2dSmemBytes == (k2dK + 3) * k2dBox * 8, "flat 2-D shared memory");

template <class GridBar>
__device__ __forceinline__ void taylor2d_body(const SolveParams& p, int border_blocks, int step, GridBar&& grid_bar) {
    if (step < 0) step = __ldcg(&p.ctrl->step);  // graph replay: the step lives on the device
    __shared__ Smem sm;
    extern __shared__ __align__(128) unsigned char dyn[];
    Ctrl* ctrl = p.ctrl;
    if (ctrl->status) return;
    trace_mark(p, kTrTaylorIn);
    const StencilOp& op = p.op;
    block_setup(p, sm, false);
    double* XS = reinterpret_cast<double*>(dyn);  // X, then T_1 .. T_{K-1}, w, -cnt, b/gamma
    double* TS = XS + k2dBox;
    double* WS = TS + (k2dK - 1) * k2dBox;
    double* NCS = WS + k2dBox;
    double* BS = NCS + k2dBox;
    const int tid = threadIdx.x, nth = blockDim.x;
    const bool leader = vcta() == 0 && tid == 0;
    gs_step_info* info = (p.infos && leader) ? p.infos + step : nullptr;
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
            sweep_l1(op, G, nullptr, nullptr, sm.wtab, [&](int64_t v, double acc, double b, double, double) {
                INC[v] = __dadd_rn(b, __dmul_rn(ht, acc));
            });
        }
        return;
    }

    // bordered column norm and (s, m): as taylor_body
    double norm_tA;
    if (bordered) {
        const bool exact = p.seq_exact && (p.infos || __ldcg(&ctrl->coln_need));
        const double coln = exact ? __ldcg(&ctrl->seq[1]) : grid_sum(p.part_c, border_blocks, sm);
        norm_tA = __dmul_rn(fabs(t), nan_dropping_max(p.anorm, coln));  // sparse.cpp:39-40
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

    // this CTA's box: the tile at (x0, y0) with a K-voxel halo; box point e = r * P + c is grid
    // point (x0 - K + c, y0 - K + r)
    const int nx = op.nx, ny = op.ny;
    const int tiles_x = (nx + k2dT - 1) / k2dT;
    const int x0 = (vcta() % tiles_x) * k2dT, y0 = (vcta() / tiles_x) * k2dT;
    auto grid_index = [&](int e) -> int64_t {
        const int x = x0 - k2dK + e % k2dP, y = y0 - k2dK + e / k2dP;
        return (x >= 0 && x < nx && y >= 0 && y < ny) ? x + static_cast<int64_t>(y) * nx : -1;
    };
    // w, -cnt and b/gamma over the box; outside the grid w = 0 (a dead row: T_k = 0, which is
    // what a missing neighbour contributes) and b/gamma = 0
    for (int e = tid; e < k2dBox; e += nth) {
        const int x = x0 - k2dK + e % k2dP, y = y0 - k2dK + e / k2dP;
        const int64_t v = grid_index(e);
        const int cnt = (x > 0) + (x < nx - 1) + (y > 0) + (y < ny - 1);
        WS[e] = v >= 0 ? sm.wtab[op.pal[v]] : 0.0;
        BS[e] = v >= 0 ? G[v] : 0.0;
        NCS[e] = __dsub_rn(-static_cast<double>(cnt), 0.0);  // the TMA sweep's ncxy - dhz with dhz = 0
        XS[e] = 0.0;
    }
    if (tid < 2 * k2dK) s_max2d[tid] = 0ull;
    const int64_t N = op.n;
    // Thread t owns tile column xl and rows ry0, ry0 + 1 for the whole launch (their f and the
    // current term stay in registers, w and -cnt too); at level k < K the first n_k - 1024
    // threads also compute one point each of the rim region_k \ tile (oR[k-1], else -1).
    const int xl = tid & (k2dT - 1), ry0 = 2 * (tid / k2dT);
    const int oA = (k2dK + ry0) * k2dP + k2dK + xl, oB = oA + k2dP;
    const int gxo = x0 + xl, gyo = y0 + ry0;
    const bool inA = gxo < nx && gyo < ny, inB = gxo < nx && gyo + 1 < ny;
    const int64_t vA = gxo + static_cast<int64_t>(gyo) * nx;
    constexpr int kRimPer = ((k2dP - 2) * (k2dP - 2) - k2dT * k2dT + kSolveThreads - 1) / kSolveThreads;
    int oR[k2dK - 1][kRimPer];
#pragma unroll
    for (int k = 1; k < k2dK; ++k) {
        const int h = k2dK - k, wk = k2dP - 2 * k;
#pragma unroll
        for (int i = 0; i < kRimPer; ++i) {
            int j = tid + i * kSolveThreads, r = -1, c = -1;
            if (j < h * wk) {  // rows above the tile
                r = k + j / wk;
                c = k + j % wk;
            } else if ((j -= h * wk) < h * wk) {  // rows below
                r = k2dK + k2dT + j / wk;
                c = k + j % wk;
            } else if ((j -= h * wk) < 2 * h * k2dT) {  // columns left and right of the tile
                r = k2dK + j / (2 * h);
                const int cc = j % (2 * h);
                c = cc < h ? k + cc : k2dK + k2dT + (cc - h);
            }
            oR[k - 1][i] = r >= 0 ? r * k2dP + c : -1;
        }
    }
    // the box of `src` (global, L2) into registers, then into X (and f: a stage starts from f)
    constexpr int kBoxIt = (k2dBox + kSolveThreads - 1) / kSolveThreads;
    auto fetch_box = [&](const double* src, double (&xr)[kBoxIt]) {
#pragma unroll
        for (int it = 0; it < kBoxIt; ++it) {  // independent loads in flight
            const int e = tid + it * kSolveThreads;
            const int64_t v = e < k2dBox ? grid_index(e) : -1;
            xr[it] = v >= 0 ? __ldcg(src + v) : 0.0;
        }
    };
    auto store_box = [&](const double (&xr)[kBoxIt]) {
#pragma unroll
        for (int it = 0; it < kBoxIt; ++it) {
            const int e = tid + it * kSolveThreads;
            if (e < k2dBox) XS[e] = xr[it];
        }
        __syncthreads();
    };

    const double tau_s = __ddiv_rn(t, static_cast<double>(s_st));  // expact.cpp:73
    double prev = __ldcg(&ctrl->prev0);
    int round = 0;  // slot rotation, identical in every CTA
    int64_t total_terms = 0;
    const double* fsrc = nullptr;  // where the final f lies
#ifdef GS_2D_PROF
    if (tid == 0) {
        for (int k = 0; k < 9; ++k) s_prof[k] = 0;
        s_prof[9] = clock64();
    }
#endif
    __syncthreads();  // the tables
    const double wA = WS[oA], wB = WS[oB], ncA = NCS[oA], ncB = NCS[oB];
    double fA = 0.0, fB = 0.0;  // f on the own points
    for (int stage = 0; stage < s_st; ++stage) {
        int kind = (stage == 0 && bordered) ? k2FirstZero : (bordered ? k2FirstBorder : k2FirstPlain);
        if (stage == 0 && !bordered) {
            double xr[kBoxIt];
            fetch_box(G, xr);
            store_box(xr);
            fA = XS[oA];
            fB = XS[oB];
        }
        int used = 0;
        while (true) {
            double* cand = p.x2d + static_cast<size_t>(round & 1) * (k2dK + 1) * N;  // f after level 1..K, then T_K
            double mx[2 * k2dK];
            PROF(0)
            double tA = 0.0, tB = 0.0;  // the previous level's term on the own points
#pragma unroll
            for (int k = 1; k <= k2dK; ++k) {
                const double ck = __ddiv_rn(tau_s, static_cast<double>(used + k));  // expact.cpp:83
                const double* src = k == 1 ? XS : TS + (k - 2) * k2dBox;
                double* dst = TS + (k - 1) * k2dBox;  // (unused at k == K)
                double* fout = cand + static_cast<size_t>(k - 1) * N;
                const bool zero = k == 1 && kind == k2FirstZero, border = k == 1 && kind == k2FirstBorder;
                // A~ applied to one point of the box: the row of the TMA sweeps, z-neighbours 0.0
                auto term = [&](int o, double w, double nc, double ym, double ctr, double yp) {
                    double sacc;
                    if (zero) {
                        sacc = __dadd_rn(0.0, BS[o]);
                    } else {
                        sacc = row_apply_nc(w, w != 0.0, nc, 0.0, ym, src[o - 1], ctr, src[o + 1], yp, 0.0);
                        if (border) sacc = __dadd_rn(sacc, BS[o]);
                    }
                    return __dmul_rn(ck, sacc);
                };
                const double cA = k == 1 ? (zero ? 0.0 : src[oA]) : tA, cB = k == 1 ? (zero ? 0.0 : src[oB]) : tB;
                const double nA = term(oA, wA, ncA, zero ? 0.0 : src[oA - k2dP], cA, cB);
                const double nB = term(oB, wB, ncB, cA, cB, zero ? 0.0 : src[oB + k2dP]);
                if (k < k2dK) {
                    dst[oA] = nA;
                    dst[oB] = nB;
#pragma unroll
                    for (int i = 0; i < kRimPer; ++i) {
                        const int o = oR[k < k2dK ? k - 1 : 0][i];
                        if (o >= 0)
                            dst[o] = term(o, WS[o], NCS[o], zero ? 0.0 : src[o - k2dP], zero ? 0.0 : src[o],
                                          zero ? 0.0 : src[o + k2dP]);
                    }
                }
                tA = nA;
                tB = nB;
                fA = __dadd_rn(fA, tA);  // f += term (expact.cpp:85-87)
                fB = __dadd_rn(fB, tB);
                mx[2 * (k - 1)] = max_abs(max_abs(0.0, tA), tB);
                mx[2 * (k - 1) + 1] = max_abs(max_abs(0.0, fA), fB);
                if (inA) {
                    fout[vA] = fA;
                    if (k == k2dK) cand[static_cast<size_t>(k2dK) * N + vA] = tA;
                }
                if (inB) {
                    fout[vA + nx] = fB;
                    if (k == k2dK) cand[static_cast<size_t>(k2dK) * N + vA + nx] = tB;
                }
                if (k < k2dK) __syncthreads();
            }
            // grid maxima of the round (as the single-term path: rotating atomicMax slots)
            {
                // block maxima: non-negative doubles order as their bit patterns -- a warp max of
                // the high words, then of the low words among the lanes that hold it, then a
                // shared-memory atomicMax per warp
                const int lane = tid & 31;
                PROF(1)
#pragma unroll
                for (int q = 0; q < 2 * k2dK; ++q) {
                    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(mx[q]));
                    const unsigned hi = static_cast<unsigned>(bits >> 32);
                    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? static_cast<unsigned>(bits) : 0u);
                    if (lane == 0) atomicMax(&s_max2d[q], (static_cast<unsigned long long>(mh) << 32) | ml);
                }
                __syncthreads();
                if (tid < 2 * k2dK) {
                    const unsigned long long v = s_max2d[tid];
                    if (v) atomicMax(p.slots + kSlots2dBase + (round % 3) * kSlots2d + tid, v);
                    s_max2d[tid] = 0ull;  // for the next round (barriers in between)
                }
                PROF(2)
                grid_bar();
                PROF(3)
                trace_mark(p, kind == k2Next ? kTrFusedNext : kTrFusedFirst);
                if (leader) {
                    unsigned long long* z = p.slots + kSlots2dBase + ((round + 2) % 3) * kSlots2d;
#pragma unroll
                    for (int q = 0; q < kSlots2d; ++q) z[q] = 0ull;
                }
                const unsigned long long* sl = p.slots + kSlots2dBase + (round % 3) * kSlots2d;
#pragma unroll
                for (int q = 0; q < 2 * k2dK; ++q) mx[q] = slot_read(sl + q);
                ++round;
            }
            // the likely next X (the stage goes on: T_K) is fetched while the maxima arrive
            double xr[kBoxIt];
            fetch_box(cand + static_cast<size_t>(k2dK) * N, xr);
            PROF(4)
            // the reference's tests, term by term (expact.cpp:88-95)
            int stop = 0;
#pragma unroll
            for (int k = 1; k <= k2dK; ++k) {
                if (stop) break;
                const double cur = mx[2 * (k - 1)];
                double fn = mx[2 * (k - 1) + 1];
                if (bordered) fn = nan_dropping_max(fn, 1.0);  // f_n == 1 (expact.cpp:89)
                ++used;
                if (!isfinite(cur) || !isfinite(fn)) {  // expact.cpp:90-91
                    if (leader) {
                        ctrl->status = GS_ENUMERIC;
                        ctrl->detail = 2;
                    }
                    return;  // uniform across CTAs
                }
                if (__dadd_rn(prev, cur) <= __dmul_rn(p.tol, fn) || used == m_deg) {  // expact.cpp:93
                    prev = fn;
                    stop = k;
                } else {
                    prev = cur;
                }
            }
            PROF(5)
            if (stop == 0) {
                kind = k2Next;
                store_box(xr);  // X = T_K; f stays
                continue;
            }
            fsrc = cand + static_cast<size_t>(stop - 1) * N;
            if (stage + 1 < s_st) {  // the next stage starts from f after term `stop`
                fetch_box(fsrc, xr);
                store_box(xr);
                fA = XS[oA];
                fB = XS[oB];
            }
            break;
        }
        total_terms += used;
        if (info && stage < kMaxLoggedStages) info->terms[stage] = used;
    }
#ifdef GS_2D_PROF
    if (leader && step == 2)
        printf("flat2d rounds %d: loadbox+misc %lld levels %lld reduce %lld gridbar %lld slots %lld decide %lld\n", round,
               s_prof[0], s_prof[1], s_prof[2], s_prof[3], s_prof[4], s_prof[5]);
#endif
    // the result, explicit in F0 (this CTA's tile, which it wrote itself)
    double* F0 = p.buf[kBufF0];
    for (int e = tid; e < k2dT * k2dT; e += nth) {
        const int gx = x0 + e % k2dT, gy = y0 + e / k2dT;
        if (gx < nx && gy < ny) {
            const int64_t v = gx + static_cast<int64_t>(gy) * nx;
            F0[v] = fsrc[v];
        }
    }
    if (info) {
        info->total_terms = total_terms;
        info->reruns = 0;
    }
    if (leader) {
        ctrl->fres = kBufF0;
        ctrl->tres = -1;
        ctrl->last_terms = static_cast<int>(total_terms);
    }
    if (p.use_tma) fence_proxy_async_global();
}
