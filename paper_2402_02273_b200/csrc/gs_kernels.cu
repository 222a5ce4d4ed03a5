// gs_kernels.cu -- sm_100a kernels of the exponential-Euler hot path.
//
//   K1 material_kernel      uint8 intensity -> Material label   (imaging.cpp:65-72, 118-141)
//   K3 colsum_norm_kernel   exact ||A||_1, matrix-free          (sparse.cpp:36-40)
//   solve_kernel            persistent cooperative kernel running whole exponential-Euler
//                           steps: RHS build (K2), bordered column + (s,m) on device,
//                           the fused Taylor-term sweeps (K4) with the in-kernel
//                           termination test, and the fused update + metrics (K5).
//
// Data layout in HBM: every field is a dense x-fastest array over the grid
// (global_index, grid.hpp:53-61); the operator is never stored -- a uint8 palette index
// per voxel plus a 256-entry table of w = D/h^2 stands for assemble_diffusion's CSR.
#include <cooperative_groups.h>

#include "gs_kernels.cuh"

namespace cg = cooperative_groups;

namespace gs {

// ----------------------------------------------------------------------------------
// K1 material map
// ----------------------------------------------------------------------------------

// nearest_source (imaging.cpp:65-72): f = i*(src-1)/(n-1), s = ceil(f - 0.5), clamped.
__device__ __forceinline__ int nearest_source(int i, int n, int src) {
    if (n <= 1 || src <= 1) return 0;
    const double f = __ddiv_rn(__dmul_rn(static_cast<double>(i), static_cast<double>(src - 1)),
                               static_cast<double>(n - 1));
    int s = static_cast<int>(ceil(__dsub_rn(f, 0.5)));
    if (s < 0) s = 0;
    if (s > src - 1) s = src - 1;
    return s;
}

__global__ void material_kernel(const uint8_t* __restrict__ stack, int w, int hgt, int slices, int nx, int ny,
                                int nz, int t_air, int t_white, int t_gray, uint8_t* __restrict__ labels) {
    const int64_t n = static_cast<int64_t>(nx) * ny * nz;
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(v % nx);
        const int j = static_cast<int>((v / nx) % ny);
        const int k = static_cast<int>(v / (static_cast<int64_t>(nx) * ny));
        const int sx = nearest_source(i, nx, w);
        const int sy = nearest_source(j, ny, hgt);
        const int sz = nearest_source(k, nz, slices);
        const int px = stack[sx + static_cast<int64_t>(sy) * w + static_cast<int64_t>(sz) * w * hgt];
        // classify (imaging.cpp:118-123)
        const uint8_t lab = px <= t_air ? 0 : px <= t_white ? 1 : px <= t_gray ? 2 : 3;
        labels[v] = lab;
    }
}

__global__ void expand_palette_kernel(const uint8_t* __restrict__ pal, const double* __restrict__ dtab, int64_t n,
                                      double* __restrict__ d) {
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x)
        d[v] = dtab[pal[v]];
}

// ----------------------------------------------------------------------------------
// K3 exact 1-norm: column c sums |a_rc| over rows r = c-sz, c-sy, c-1, c, c+1, c+sy, c+sz
// in ascending r -- the CSR storage order the reference's constructor walks
// (sparse.cpp:36-38) -- so every column sum is bit-identical; the max is order-free.
// ----------------------------------------------------------------------------------
__global__ void colsum_norm_kernel(StencilOp op, unsigned long long* out_bits) {
    __shared__ double s_wtab[256];
    if (op.pal)
        for (int q = threadIdx.x; q < 256; q += blockDim.x) s_wtab[q] = op.wtab[q];
    __syncthreads();
    double best = 0.0;
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < op.n;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(c % op.nx);
        const int j = static_cast<int>((c / op.nx) % op.ny);
        const int k = static_cast<int>(c / op.sz);
        auto offw = [&](int64_t r) {
            const RowCoef rc = row_coef(op, s_wtab, r);
            return rc.live ? fabs(rc.w) : 0.0;
        };
        double s = 0.0;
        if (k > 0) s = __dadd_rn(s, offw(c - op.sz));
        if (j > 0) s = __dadd_rn(s, offw(c - op.sy));
        if (i > 0) s = __dadd_rn(s, offw(c - 1));
        {
            const RowCoef rc = row_coef(op, s_wtab, c);
            const int cnt = (i > 0) + (i < op.nx - 1) + (j > 0) + (j < op.ny - 1) + (k > 0) + (k < op.nz - 1);
            if (rc.live) s = __dadd_rn(s, fabs(__dmul_rn(static_cast<double>(-cnt), rc.w)));
        }
        if (i < op.nx - 1) s = __dadd_rn(s, offw(c + 1));
        if (j < op.ny - 1) s = __dadd_rn(s, offw(c + op.sy));
        if (k < op.nz - 1) s = __dadd_rn(s, offw(c + op.sz));
        best = nan_dropping_max(best, s);
    }
    best = warp_max(best);
    if ((threadIdx.x & 31) == 0 && best > 0.0)
        atomicMax(out_bits, static_cast<unsigned long long>(__double_as_longlong(best)));
}

// ----------------------------------------------------------------------------------
// Persistent exponential-Euler kernel
// ----------------------------------------------------------------------------------

// Work decomposition: an item is a kTX x kTY column tile times a z-chunk; a CTA walks
// items round-robin.  Each thread owns one (i, j) column of the tile and marches it
// through the chunk, carrying x(z-1), x(z), x(z+1) of its column in registers; the four
// in-plane neighbours come through L1 (the CTA reads the whole tile plane).
template <bool kStencil, class Body>
__device__ __forceinline__ void sweep(const StencilOp& op, const double* X, const double* s_wtab, Body&& body) {
    const int lx = threadIdx.x % kTX, ly = threadIdx.x / kTX;
    const int64_t tiles = static_cast<int64_t>(op.tiles_x) * op.tiles_y;
    for (int64_t item = blockIdx.x; item < op.n_items; item += gridDim.x) {
        const int64_t tile = item % tiles;
        const int chunk = static_cast<int>(item / tiles);
        const int i = static_cast<int>(tile % op.tiles_x) * kTX + lx;
        const int j = static_cast<int>(tile / op.tiles_x) * kTY + ly;
        const bool act = i < op.nx && j < op.ny;
        const int z0 = chunk * op.zc;
        const int z1 = min(op.nz, z0 + op.zc);
        const int64_t colv = i + static_cast<int64_t>(j) * op.sy;
        double xm = 0.0, xc = 0.0;
        if (kStencil && act) {
            xm = z0 > 0 ? X[colv + (z0 - 1) * op.sz] : 0.0;
            xc = X[colv + z0 * op.sz];
        }
        const bool hx0 = i > 0, hx1 = i < op.nx - 1, hy0 = j > 0, hy1 = j < op.ny - 1;
        for (int k = z0; k < z1; ++k) {
            const int64_t v = colv + k * op.sz;
            double acc = 0.0;
            if (kStencil) {
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
                    acc = row_apply(rc, cnt, xm, xym, xxm, xc, xxp, xyp, xp);
                }
                xm = xc;
                xc = xp;
            }
            if (act) body(v, i, j, k, acc);
        }
    }
}

struct Smem {
    double wtab[256];
    double red[kThreads / 32][4];
    double bcast[4];
};

// Block reduction of up to 4 values with a fixed shape; result valid in thread 0.
template <int K, bool kMax>
__device__ __forceinline__ void block_reduce(double (&v)[K], Smem& sm) {
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
            for (int w = 1; w < kThreads / 32; ++w) a = kMax ? nan_dropping_max(a, sm.red[w][q]) : __dadd_rn(a, sm.red[w][q]);
            v[q] = a;
        }
    }
    __syncthreads();
}

// Deterministic sum of the per-CTA partials; every CTA computes the same value.
__device__ double grid_sum(const double* part, int nb, Smem& sm) {
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

enum TermKind { kFirstZero, kFirstBorder, kFirstPlain, kNext };

__global__ void __launch_bounds__(kThreads) solve_kernel(const __grid_constant__ SolveParams p) {
    cg::grid_group grid = cg::this_grid();
    __shared__ Smem sm;
    const StencilOp& op = p.op;
    if (op.pal)
        for (int q = threadIdx.x; q < 256; q += kThreads) sm.wtab[q] = __ldg(op.wtab + q);
    __syncthreads();
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    int round = 0;  // per-term max-reduction rounds (slot rotation, identical in every CTA)

    auto sync_round = [&]() {
        grid.sync();
        if (leader) {
            unsigned long long* z = p.slots + ((round + 2) % 3) * 4;
            z[0] = z[1] = z[2] = z[3] = 0ull;
        }
        ++round;
    };
    auto push_max2 = [&](double a, double b) {
        double v[2] = {a, b};
        block_reduce<2, true>(v, sm);
        if (threadIdx.x == 0) {
            unsigned long long* s = p.slots + (round % 3) * 4;
            if (v[0] > 0.0) atomicMax(s + 0, static_cast<unsigned long long>(__double_as_longlong(v[0])));
            if (v[1] > 0.0) atomicMax(s + 1, static_cast<unsigned long long>(__double_as_longlong(v[1])));
        }
    };

    // compute_metrics (integrator.cpp:65-89) of p.u: sum in a fixed tree (the reference's
    // serial sum differs in the last bits), max/min/front radius exactly.
    auto metrics_local = [&](double& sum, double& mx, double& mn, double& r2, int64_t v, int i, int j, int k,
                             double u) {
        sum = __dadd_rn(sum, u);
        mx = nan_dropping_max(mx, u);
        mn = (u < mn) ? u : mn;
        if (u >= p.front_threshold) {
            const double dx = __dsub_rn(__dadd_rn(p.origin[0], __dmul_rn(static_cast<double>(i), p.h)), p.center[0]);
            const double dy = __dsub_rn(__dadd_rn(p.origin[1], __dmul_rn(static_cast<double>(j), p.h)), p.center[1]);
            const double dz = __dsub_rn(__dadd_rn(p.origin[2], __dmul_rn(static_cast<double>(k), p.h)), p.center[2]);
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            r2 = nan_dropping_max(r2, d2);
        }
        (void)v;
    };
    auto metrics_push = [&](double sum, double mx, double mn, double r2, int parity) {
        double s[1] = {sum};
        block_reduce<1, false>(s, sm);
        if (threadIdx.x == 0) p.part_u[blockIdx.x] = s[0];
        // max / min / r2 through order-free atomics on ordered keys
        const double mxw = warp_max(mx);
        double mnw = mn;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double q = __shfl_xor_sync(0xffffffffu, mnw, o);
            mnw = (q < mnw) ? q : mnw;
        }
        const double r2w = warp_max(r2);
        if ((threadIdx.x & 31) == 0) {
            unsigned long long* ms = p.mslots + parity * 4;
            atomicMax(ms + 0, ordered_key(mxw));
            atomicMin(ms + 1, ordered_key(mnw));
            if (r2w > 0.0) atomicMax(ms + 2, static_cast<unsigned long long>(__double_as_longlong(r2w)));
        }
    };
    // After the barrier that follows metrics_push: the leader records node `node`.
    auto metrics_finish = [&](int node, int parity) {
        const double sum = grid_sum(p.part_u, p.grid_blocks, sm);
        if (leader) {
            unsigned long long* ms = p.mslots + parity * 4;
            const double cell = __dmul_rn(__dmul_rn(p.h, p.h), p.h);
            double* out = p.metrics + 4 * node;
            out[0] = __dmul_rn(cell, sum);
            out[1] = from_ordered_key(__ldcg(ms + 0));
            out[2] = from_ordered_key(__ldcg(ms + 1));
            out[3] = sqrt(__longlong_as_double(static_cast<long long>(__ldcg(ms + 2))));
            ms[0] = 0ull;
            ms[1] = ~0ull;
            ms[2] = 0ull;
        }
    };

    // -------------------------------------------------------------- y = A x
    if (p.mode == kModeApply) {
        sweep<true>(op, p.g, sm.wtab, [&](int64_t v, int, int, int, double acc) { p.out[v] = acc; });
        return;
    }

    const bool run = p.mode == kModeRun;
    const bool bordered = p.mode != kModeExpmv;
    const double t = p.tau;

    if (run && p.want_metrics) {
        double sum = 0.0, mx = -INFINITY, mn = INFINITY, r2 = 0.0;
        sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int i, int j, int k, double) {
            metrics_local(sum, mx, mn, r2, v, i, j, k, p.u[v]);
        });
        metrics_push(sum, mx, mn, r2, 0);
        grid.sync();
        metrics_finish(0, 0);
    }

    const int n_steps = run ? p.n_steps : 1;
    for (int step = 0; step < n_steps; ++step) {
        gs_step_info* info = (p.infos && leader) ? p.infos + step : nullptr;
        if (info) {
            info->s = info->m = 1;
            info->branch = 0;
            info->total_terms = 0;
            info->anorm = p.anorm;
            info->bnorm = info->coln = info->gamma = info->norm_tA = 0.0;
        }
        double* G = p.g;
        double bnorm = 0.0;
        // ---------------------------------------------------------- K2: RHS + ||b||_1
        if (run) {
            // g = A u; g += rho*u*(1-u)   (integrator.cpp:54-57)
            double bsum = 0.0;
            sweep<true>(op, p.u, sm.wtab, [&](int64_t v, int, int, int, double acc) {
                const double u = p.u[v];
                const double g = __dadd_rn(acc, __dmul_rn(__dmul_rn(p.rho, u), __dsub_rn(1.0, u)));
                G[v] = g;
                bsum = __dadd_rn(bsum, fabs(g));
            });
            double s[1] = {bsum};
            block_reduce<1, false>(s, sm);
            if (threadIdx.x == 0) p.part_b[blockIdx.x] = s[0];
        } else if (bordered) {
            double bsum = 0.0;
            sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int, int, int, double) {
                bsum = __dadd_rn(bsum, fabs(G[v]));
            });
            double s[1] = {bsum};
            block_reduce<1, false>(s, sm);
            if (threadIdx.x == 0) p.part_b[blockIdx.x] = s[0];
        } else {
            // expmv: prev = ||b||_inf at stage 0 (expact.cpp:80)
            double mb = 0.0;
            sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int, int, int, double) {
                mb = nan_dropping_max(mb, fabs(G[v]));
            });
            push_max2(mb, 0.0);
        }
        grid.sync();

        double* Fcur = nullptr;
        double scale = 0.0;
        int branch = 0;
        double prev0 = 1.0;  // ||e_{n+1}||_inf for the bordered action
        if (bordered) {
            bnorm = grid_sum(p.part_b, p.grid_blocks, sm);
            if (info) info->bnorm = bnorm;
            if (t == 0.0) branch = 1;                                  // expact.cpp:108
            else if (bnorm == 0.0) branch = 2;                         // expact.cpp:111
            else if (__dmul_rn(fabs(t), p.anorm) <= 1e-8) branch = 3;  // expact.cpp:114
        } else {
            prev0 = slot_read(p.slots + (round % 3) * 4);
            if (leader) {
                unsigned long long* z = p.slots + ((round + 2) % 3) * 4;
                z[0] = z[1] = z[2] = z[3] = 0ull;
            }
            ++round;
        }
        if (info) info->branch = branch;

        if (branch != 0) {
            // phi1v degenerate branches, then the step update u + tau*incr
            if (branch == 3) {
                // incr = b + 0.5*t*(A b)   (expact.cpp:117-121)
                const double ht = __dmul_rn(0.5, t);
                sweep<true>(op, G, sm.wtab, [&](int64_t v, int, int, int, double acc) {
                    const double incr = __dadd_rn(G[v], __dmul_rn(ht, acc));
                    if (run) p.t[0][v] = incr;
                    else p.out[v] = incr;
                });
                if (run) {
                    grid.sync();  // A*G read G's neighbours; the update below is pointwise
                }
            }
            if (run) {
                double sum = 0.0, mx = -INFINITY, mn = INFINITY, r2 = 0.0;
                sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int i, int j, int k, double) {
                    const double incr = branch == 1 ? G[v] : branch == 2 ? 0.0 : p.t[0][v];
                    const double un = __dadd_rn(p.u[v], __dmul_rn(t, incr));
                    p.u[v] = un;
                    if (p.want_metrics) metrics_local(sum, mx, mn, r2, v, i, j, k, un);
                });
                if (p.want_metrics) metrics_push(sum, mx, mn, r2, (step + 1) & 1);
                grid.sync();
                if (p.want_metrics) metrics_finish(step + 1, (step + 1) & 1);
            } else if (branch != 3) {
                sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int, int, int, double) {
                    p.out[v] = branch == 1 ? G[v] : 0.0;
                });
            }
            continue;
        }

        // ------------------------------------------- bordered column b/gamma and (s, m)
        double gamma = 0.0, norm_tA;
        if (bordered) {
            gamma = __ddiv_rn(bnorm, p.anorm);  // expact.cpp:126
            double csum = 0.0;
            sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int, int, int, double) {
                const double b = G[v];
                const double bg = (b != 0.0) ? __ddiv_rn(b, gamma) : 0.0;  // expact.cpp:137-138
                G[v] = bg;
                csum = __dadd_rn(csum, fabs(bg));
            });
            double s[1] = {csum};
            block_reduce<1, false>(s, sm);
            if (threadIdx.x == 0) p.part_c[blockIdx.x] = s[0];
            grid.sync();
            const double coln = grid_sum(p.part_c, p.grid_blocks, sm);
            // bordered ||.||_1 = max over columns: A's columns, then column n (sparse.cpp:39-40)
            norm_tA = __dmul_rn(fabs(t), nan_dropping_max(p.anorm, coln));
            if (info) {
                info->coln = coln;
                info->gamma = gamma;
            }
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
                p.status[0] = sel;
                p.status[1] = 1;  // select_params
            }
            return;  // uniform across CTAs
        }

        // ------------------------------------------------------------- K4: Taylor terms
        const double tau_s = __ddiv_rn(t, static_cast<double>(s_st));  // expact.cpp:73
        Fcur = bordered ? nullptr : G;  // nullptr: f = e_{n+1} (all zero) for the bordered action
        const double* Tprev = nullptr;
        int fsel = 0, tsel = 0;
        double prev = prev0;
        int64_t total_terms = 0;
        for (int stage = 0; stage < s_st; ++stage) {
            int used = 0;
            for (int j = 1; j <= m_deg; ++j) {
                const double c = __ddiv_rn(tau_s, static_cast<double>(j));  // expact.cpp:83
                const TermKind kind = j > 1 ? kNext : (Fcur == nullptr ? kFirstZero : (bordered ? kFirstBorder : kFirstPlain));
                double* Fout = p.f[fsel];
                double* Tout = p.t[tsel];
                double mt = 0.0, mf = 0.0;
                // term = c * (A~ term); f += term   (expact.cpp:82-87)
                if (kind == kFirstZero) {
                    sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int, int, int, double) {
                        const double tn = __dmul_rn(c, __dadd_rn(0.0, G[v]));
                        const double fn = __dadd_rn(0.0, tn);
                        Tout[v] = tn;
                        Fout[v] = fn;
                        mt = nan_dropping_max(mt, fabs(tn));
                        mf = nan_dropping_max(mf, fabs(fn));
                    });
                } else {
                    const double* X = (kind == kNext) ? Tprev : Fcur;
                    const double* Fin = Fcur;
                    sweep<true>(op, X, sm.wtab, [&](int64_t v, int, int, int, double acc) {
                        // the border entry (column n, value b_i/gamma) is the last in its row and
                        // term_n = 1 only on a stage's first term (expact.cpp:137-138, :96)
                        const double sc = (kind == kFirstBorder) ? __dadd_rn(acc, G[v]) : acc;
                        const double tn = __dmul_rn(c, sc);
                        const double fn = __dadd_rn(Fin[v], tn);
                        Tout[v] = tn;
                        Fout[v] = fn;
                        mt = nan_dropping_max(mt, fabs(tn));
                        mf = nan_dropping_max(mf, fabs(fn));
                    });
                }
                push_max2(mt, mf);
                sync_round();
                ++used;
                Fcur = Fout;
                Tprev = Tout;
                fsel ^= 1;
                tsel ^= 1;
                const unsigned long long* sl = p.slots + ((round - 1) % 3) * 4;
                const double cur = slot_read(sl + 0);
                double fnorm = slot_read(sl + 1);
                if (bordered) fnorm = nan_dropping_max(fnorm, 1.0);  // f_n == 1 (expact.cpp:89)
                if (!isfinite(cur) || !isfinite(fnorm)) {             // expact.cpp:90-91
                    if (leader) {
                        p.status[0] = GS_ENUMERIC;
                        p.status[1] = 2;
                    }
                    return;
                }
                if (__dadd_rn(prev, cur) <= __dmul_rn(p.tol, fnorm)) {  // expact.cpp:93
                    prev = fnorm;  // next stage: term = f, ||term|| = ||f|| (expact.cpp:80, :96)
                    break;
                }
                prev = cur;
                if (j == m_deg) {
                    prev = fnorm;
                }
            }
            total_terms += used;
            if (info && stage < kMaxLoggedStages) info->terms[stage] = used;
        }
        if (info) info->total_terms = total_terms;

        // ------------------------------------------------ K5: output / update + metrics
        if (run) {
            const double scl = __ddiv_rn(gamma, t);  // expact.cpp:150
            double sum = 0.0, mx = -INFINITY, mn = INFINITY, r2 = 0.0;
            const double* F = Fcur;
            sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int i, int j, int k, double) {
                // out = u + tau * (scale * y)   (integrator.cpp:59-61, expact.cpp:151)
                const double un = __dadd_rn(p.u[v], __dmul_rn(t, __dmul_rn(scl, F[v])));
                p.u[v] = un;
                if (p.want_metrics) metrics_local(sum, mx, mn, r2, v, i, j, k, un);
            });
            if (p.want_metrics) metrics_push(sum, mx, mn, r2, (step + 1) & 1);
            grid.sync();
            if (p.want_metrics) metrics_finish(step + 1, (step + 1) & 1);
        } else {
            scale = bordered ? __ddiv_rn(gamma, t) : 1.0;
            const double* F = Fcur;
            sweep<false>(op, nullptr, sm.wtab, [&](int64_t v, int, int, int, double) {
                p.out[v] = bordered ? __dmul_rn(scale, F[v]) : F[v];
            });
        }
    }
}

}  // namespace gs
