// gs_seqsum.cuh -- the reference's SEQUENTIAL sums of |x_i|, reproduced bit for bit in parallel.
//
// Two sums on the path are order-dependent:
//   ||b||_1 = sum_i |b_i|                  one_norm (expact.cpp:20-24), called at expact.cpp:110
//   colsum[n] = sum_{b_i != 0} |b_i/gamma| the bordered column of the operator's constructor
//                                          (sparse.cpp:36-38 on the CSR built at expact.cpp:131-142)
// both a plain left-to-right loop s = fl(s + x_i) over i = 0..n-1.  A tree sum differs from it
// in the last bits, and at some configurations (2-D C2, s = 10 stages) one ulp of ||b||_1 moves
// the step's u by 1e-10 relative: the reference's phi1v is that sensitive to gamma.  So the
// device computes exactly the sequential value.
//
// Why that is parallel: all x_i >= 0, so the partial sums s_i are non-decreasing.  While s stays
// in one binade [2^B, 2^(B+1)) every s_i is an integer multiple m_i of u = 2^(B-52), and
// fl(s + x) = (m + r(x, parity(m))) u with r = x/u rounded to nearest (ties: to even m + r) --
// an integer increment that depends on s only through the parity of m.  A run of elements in
// one binade therefore has a summary (d0, d1) = total increment for an even / odd starting m,
// and summaries compose associatively (pcompose).  Only the elements at which s changes binade
// (a few hundred: s climbs from the tails of the Gaussian to O(1)) need a real fl(s + x).
//
// Plan (per run, i.e. per member of an ensemble; cpm CTAs = its virtual grid):
//   seqsum_tiles: tiles of kSeqTile elements; an approximate sum per tile (any order), the
//                 non-finite flags; the last CTA turns them into approximate exclusive prefixes.
//   seqsum_items: each CTA walks a contiguous range of tiles.  The approximate prefix a_i
//                 (error << delta) predicts each element's binade: an element is "clean" when
//                 a_i (1-delta) and (a_i + x_i)(1+delta) share a binade B_i, else "raw".
//                 Maximal runs of clean elements with one B become items (B, d0, d1, start,
//                 len); raw elements become items of their own.  A block-wide segmented scan
//                 builds them; the CTA appends them to its list.  The last CTA to finish walks
//                 all lists in order from s = 0: a run is applied as m += d[m & 1] after
//                 checking that s really is in binade B and stays in it (m + d <= 2^53); a raw
//                 item, or a run whose check fails, is added element by element with __dadd_rn.
// The checks make the result exact whatever the prediction: the prediction only decides how
// much of the walk is O(1) per run.

namespace seq {

constexpr uint64_t kM52 = (1ull << 52) - 1;
constexpr uint64_t kTwo52 = 1ull << 52;
constexpr uint64_t kTwo53 = 1ull << 53;
constexpr uint64_t kSat = 1ull << 62;  // saturated increment: "leaves the binade"
constexpr double kDelta = 0x1p-24;     // prefix-prediction margin (>> n * 2^-53 for n < 2^28)

enum Kind : int { kEmpty = 0, kRun = 1, kRaw = 2, kMixed = 3 };
enum Flag : unsigned { kHasNaN = 1u, kHasInf = 2u };

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b) {
    const uint64_t s = a + b;  // a, b <= kSat: no wrap
    return s > kSat ? kSat : s;
}

// Binade of a finite s >= 0: s is a multiple of 2^(B-52) (subnormals and [2^-1022, 2^-1021)
// share B = -1022).
__device__ __forceinline__ int binade(double s) {
    const int e = static_cast<int>(static_cast<unsigned long long>(__double_as_longlong(s)) >> 52);
    return (e > 0 ? e : 1) - 1023;
}

struct Pair {
    uint64_t d0, d1;  // increment in units of 2^(B-52) from an even / an odd multiple
};

// a then b
__device__ __forceinline__ Pair pcompose(const Pair& a, const Pair& b) {
    const uint64_t b0 = (a.d0 & 1) ? b.d1 : b.d0;
    const uint64_t b1 = (a.d1 & 1) ? b.d0 : b.d1;  // parity after a from an odd m: (1 + a.d1) & 1
    return {sat_add(a.d0, b0), sat_add(a.d1, b1)};
}

// The increment of fl(s + x) on the grid 2^(B-52) for 0 <= x finite: x = mx 2^ex exactly, so
// x / u = mx 2^sh; round to nearest, ties to the even result (which depends on m's parity).
__device__ __forceinline__ Pair elem_pair(double x, int B) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
    const int ex = static_cast<int>(bits >> 52);
    const uint64_t mx = (bits & kM52) | (ex ? kTwo52 : 0ull);
    if (mx == 0) return {0, 0};
    const int sh = (ex ? ex : 1) - 1075 - (B - 52);
    if (sh >= 0) {
        if (sh >= 62 || (mx >> (62 - sh)) != 0) return {kSat, kSat};
        const uint64_t k = mx << sh;
        return {k, k};
    }
    const int n = -sh;
    if (n >= 64) return {0, 0};  // x < u/2^11: half > mx, absorbed
    const uint64_t k = mx >> n, rem = mx & ((1ull << n) - 1), half = 1ull << (n - 1);
    const uint64_t r0 = k + (rem > half ? 1ull : 0ull);
    if (rem != half) return {r0, r0};
    return (k & 1) ? Pair{r0 + 1, r0} : Pair{r0, r0 + 1};  // tie: round to the even m + r
}

// The fast path's element increment without the parity rule: x/u rounded half-down, with
// `tie` set when x/u is exactly halfway (then only the parity-tracking pair path is exact) and
// `big` when x reaches 2^53 u (the element cannot belong to a run of binade B).
__device__ __forceinline__ uint64_t elem_r0(double x, int B, bool& tie, bool& big) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
    const int ex = static_cast<int>(bits >> 52);
    const uint64_t mx = (bits & kM52) | (ex ? kTwo52 : 0ull);
    const int sh = (ex ? ex : 1) - 1075 - (B - 52);
    if (sh >= 0) {
        big = big || (mx != 0 && (sh >= 1 || mx >= kTwo53));
        return mx;  // (only meaningful when !big: sh == 0)
    }
    const int n = -sh;
    if (n >= 64) return 0;
    const uint64_t half = 1ull << (n - 1), rem = mx & ((1ull << n) - 1);
    tie = tie || rem == half;
    return (mx + half - 1) >> n;  // k + (rem > half)
}

// s <- s + run, when s is in binade B and the run keeps it there; false otherwise.
__device__ __forceinline__ bool apply_run(double& s, int B, const Pair& d) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
    const int e = static_cast<int>(bits >> 52);
    if ((e > 0 ? e : 1) - 1023 != B) return false;
    const uint64_t m = (bits & kM52) | (e ? kTwo52 : 0ull);
    const uint64_t mm = m + ((m & 1) ? d.d1 : d.d0);
    if (mm > kTwo53) return false;
    uint64_t ob;
    if (mm == kTwo53) ob = static_cast<uint64_t>(B + 1 + 1023) << 52;  // exactly 2^(B+1) (B+1 = 1024: inf)
    else if (mm < kTwo52) ob = mm;                                     // subnormal (B = -1022 only)
    else ob = (static_cast<uint64_t>(B + 1023) << 52) | (mm & kM52);
    s = __longlong_as_double(static_cast<long long>(ob));
    return true;
}

// A segment of the element sequence: empty, a clean run in one binade, one raw element
// (d.d0 = its bits), or a mixed run (an inconsistency: walked element by element).
struct Seg {
    int kind, B;
    Pair d;
    int64_t start;
};

__device__ __forceinline__ Seg seg_combine(const Seg& a, const Seg& b) {
    if (a.kind == kEmpty) return b;
    if (b.kind == kEmpty) return a;
    Seg r = a;
    if (a.kind == kRun && b.kind == kRun && a.B == b.B) r.d = pcompose(a.d, b.d);
    else r.kind = kMixed;
    return r;
}

struct Item {
    int kind, B;
    uint64_t d0, d1;
    int64_t start, len;
};

__device__ __forceinline__ Seg shfl_up_seg(const Seg& v, int o) {
    Seg r;
    const long long kb = (static_cast<long long>(v.kind) << 32) | static_cast<unsigned>(v.B);
    const long long kb2 = __shfl_up_sync(0xffffffffu, kb, o);
    r.kind = static_cast<int>(kb2 >> 32);
    r.B = static_cast<int>(static_cast<unsigned>(kb2));
    r.d.d0 = __shfl_up_sync(0xffffffffu, v.d.d0, o);
    r.d.d1 = __shfl_up_sync(0xffffffffu, v.d.d1, o);
    r.start = __shfl_up_sync(0xffffffffu, v.start, o);
    return r;
}

// op((fa, a), (fb, b)) = (fa | fb, fb ? b : a + b): segmented scan, a before b
__device__ __forceinline__ void seg_op(bool fa, const Seg& a, bool& fb, Seg& b) {
    if (!fb) b = seg_combine(a, b);
    fb = fb || fa;
}

// Does any value of the bordered column sum within the tree sum's error bound give the same
// select_params (expact.cpp:29-61) result?  The sequential and the tree sums of the same n
// non-negative values both lie within (n-1) 2^-53 (relative) of the true sum, so the sequential
// one lies in [lo, hi] below.  select_params depends on the norm only through
// stages(m) = max(1, ceil(norm / r_m)), monotone in the norm: if every m has the same stage
// count at both ends, the whole interval -- the exact value included -- selects the same
// (s, m).  Then only the reported value needs the exact sum.
__device__ __forceinline__ bool coln_settles(double t, double anorm, double coln_tree, int64_t n, const double* rtab,
                                             int max_degree) {
    if (!isfinite(coln_tree)) return false;
    const double e = static_cast<double>(n + 64) * 0x1p-52;
    const double lo = __dmul_rn(coln_tree, 1.0 - e), hi = __dmul_rn(coln_tree, 1.0 + e);
    const double nlo = __dmul_rn(fabs(t), anorm < lo ? lo : anorm);
    const double nhi = __dmul_rn(fabs(t), anorm < hi ? hi : anorm);
    if (!isfinite(nhi)) return false;
    for (int m = 1; m <= max_degree; ++m)
        if (ceil(__ddiv_rn(nlo, rtab[m])) != ceil(__ddiv_rn(nhi, rtab[m]))) return false;
    return true;
}

}  // namespace seq

// The walk's state: s = m 2^(B-52) with m < 2^53 (s = 0: B = -1022, m = 0).
struct SeqState {
    int B;
    uint64_t m;
    __device__ __forceinline__ double value() const {
        const uint64_t bits = m < seq::kTwo52 ? m : ((static_cast<uint64_t>(B + 1023) << 52) | (m & seq::kM52));
        return __longlong_as_double(static_cast<long long>(bits));
    }
    __device__ __forceinline__ void set(double s) {  // finite s >= 0
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
        const int e = static_cast<int>(bits >> 52);
        B = (e > 0 ? e : 1) - 1023;
        m = (bits & seq::kM52) | (e ? seq::kTwo52 : 0ull);
    }
};

constexpr int kSeqEPT = 8;                          // elements per thread and tile
constexpr int kSeqTile = kSolveThreads * kSeqEPT;   // elements per tile
constexpr int kSeqItemCap = 512;                    // items per CTA list

struct SeqSmem {
    double dred[kSolveThreads / 32];
    int ired[kSolveThreads / 32];
    seq::Seg wseg[kSolveThreads / 32];
    seq::Pair wpair[2][kSolveThreads / 32];  // fast tiles' warp summaries, double-buffered
    bool wflag[kSolveThreads / 32];
    int lastB[kSolveThreads];      // per thread: binade of its last element (-2000: raw)
    seq::Seg open;                 // the CTA's open segment carried across its tiles
    int open_B;                    // binade of the previous element (-2000: raw / none)
    int items;                     // items emitted so far
    bool last, fin;
    double bcast;
    SeqState st;  // the composer's walk state between item batches
};

// Exclusive block scan of doubles (fixed order); also returns the block total in *total.
__device__ __forceinline__ double seq_block_excl_sum(double v, SeqSmem& sm, double* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = __dadd_rn(y, inc);
    }
    double ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0.0;
    if (lane == 31) sm.dred[w] = inc;
    __syncthreads();
    double carry = 0.0, tot = 0.0;
    for (int q = 0; q < kSolveThreads / 32; ++q) {
        if (q == w) carry = tot;
        tot = __dadd_rn(tot, sm.dred[q]);
    }
    __syncthreads();
    if (total) *total = tot;
    return __dadd_rn(carry, ex);
}

__device__ __forceinline__ int seq_block_excl_int(int v, SeqSmem& sm, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    int ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0;
    if (lane == 31) sm.ired[w] = inc;
    __syncthreads();
    int carry = 0, tot = 0;
    for (int q = 0; q < kSolveThreads / 32; ++q) {
        if (q == w) carry = tot;
        tot += sm.ired[q];
    }
    __syncthreads();
    if (total) *total = tot;
    return carry + ex;
}

constexpr int kSeqRawB = -3000, kSeqPadB = -4000, kSeqStartB = -5000;

// Reset the CTA's open segment before the first tile of a contiguous range (thread 0; the
// caller synchronises).
__device__ __forceinline__ void seq_open_reset(SeqSmem& sm) {
    sm.items = 0;
    sm.open = seq::Seg{seq::kEmpty, 0, {0, 0}, 0};
    sm.open_B = kSeqStartB;
}

// The items of one tile: elements e = 0 .. cnt-1 at X[e] (global index base + e), thread t
// owning e in [t EPT, t EPT + EPT); a_tile approximates the sequential sum before the tile.
// Items go to items[sm.items ..] (up to cap; sm.items counts past it on overflow); the open
// segment carries over to the next tile in sm.  Every thread of the block must call it.
template <int EPT>
__device__ __forceinline__ void seq_tile_items(SeqSmem& sm, const double (&xin)[EPT], int64_t base, int cnt,
                                               double a_tile, seq::Item* items, int cap) {
    using seq::Seg;
    const int e0 = static_cast<int>(threadIdx.x) * EPT;
    double x[EPT];
    double ts = 0.0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        x[j] = e0 + j < cnt ? fabs(xin[j]) : 0.0;
        ts = __dadd_rn(ts, x[j]);
    }
    double tile_sum;
    const double a0 = __dadd_rn(a_tile, seq_block_excl_sum(ts, sm, &tile_sum));
    // Fast path: the whole tile stays in one binade (its approximate prefix interval, widened
    // by delta, does) -- one run: an ordered block reduction of the element summaries, merged
    // into the CTA's open segment.  Block-uniform: a_tile and tile_sum are.
    {
        const int bt = seq::binade(__dmul_rn(a_tile, 1.0 - seq::kDelta));
        const double a_end = __dmul_rn(__dadd_rn(a_tile, tile_sum), 1.0 + seq::kDelta);
        if (cnt > 0 && isfinite(a_end) && bt == seq::binade(a_end)) {
            seq::Pair d{0, 0};
#pragma unroll
            for (int j = 0; j < EPT; ++j)
                if (e0 + j < cnt) d = seq::pcompose(d, seq::elem_pair(x[j], bt));
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {  // ordered: lane l absorbs lane l + o
                const uint64_t q0 = __shfl_down_sync(0xffffffffu, d.d0, o);
                const uint64_t q1 = __shfl_down_sync(0xffffffffu, d.d1, o);
                if ((lane & (2 * o - 1)) == 0) d = seq::pcompose(d, seq::Pair{q0, q1});
            }
            if (lane == 0) sm.wseg[w].d = d;
            __syncthreads();
            if (threadIdx.x == 0) {
                seq::Pair t{0, 0};
                for (int q = 0; q < kSolveThreads / 32; ++q) t = seq::pcompose(t, sm.wseg[q].d);
                Seg& o = sm.open;
                if (o.kind == seq::kRun && o.B == bt && sm.open_B == bt) {
                    o.d = seq::pcompose(o.d, t);
                } else {
                    if (o.kind != seq::kEmpty) {
                        if (sm.items < cap) items[sm.items] = seq::Item{o.kind, o.B, o.d.d0, o.d.d1, o.start, base - o.start};
                        ++sm.items;
                    }
                    o = Seg{seq::kRun, bt, t, base};
                }
                sm.open_B = bt;
            }
            __syncthreads();
            return;
        }
    }
    // predicted binade of every element (kSeqRawB: the prefix may change binade at it)
    int bj[EPT];
    double a = a0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const double an = __dadd_rn(a, x[j]);
        const int bl = seq::binade(__dmul_rn(a, 1.0 - seq::kDelta));
        const int bh = seq::binade(__dmul_rn(an, 1.0 + seq::kDelta));
        bj[j] = e0 + j >= cnt ? kSeqPadB : (bl == bh ? bl : kSeqRawB);
        a = an;
    }
    sm.lastB[threadIdx.x] = bj[EPT - 1];
    __syncthreads();
    const int prevB0 = threadIdx.x ? sm.lastB[threadIdx.x - 1] : sm.open_B;
    auto value = [&](int j) -> Seg {
        const int64_t i = base + e0 + j;
        if (bj[j] == kSeqRawB) return Seg{seq::kRaw, 0, {static_cast<uint64_t>(__double_as_longlong(x[j])), 0}, i};
        return Seg{seq::kRun, bj[j], seq::elem_pair(x[j], bj[j]), i};
    };
    // pass A: starts among this thread's elements, and the segment open after the last one
    bool hs = false;
    int ns = 0;
    Seg cur{seq::kEmpty, 0, {0, 0}, 0};
    int pb = prevB0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        if (bj[j] == kSeqPadB) break;
        const Seg v = value(j);
        if (bj[j] != pb || bj[j] == kSeqRawB) {
            hs = true;
            ++ns;
            cur = v;
        } else {
            cur = seq::seg_combine(cur, v);
        }
        pb = bj[j];
    }
    // block-wide segmented exclusive scan of (hs, cur); carry-in: the CTA's open segment
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    bool f = hs;
    Seg v = cur;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const bool fo = __shfl_up_sync(0xffffffffu, f, o);
        const Seg vo = seq::shfl_up_seg(v, o);
        if (lane >= o) seq::seg_op(fo, vo, f, v);
    }
    bool fe = __shfl_up_sync(0xffffffffu, f, 1);
    Seg ve = seq::shfl_up_seg(v, 1);
    if (lane == 0) {
        fe = false;
        ve = Seg{seq::kEmpty, 0, {0, 0}, 0};
    }
    if (lane == 31) {
        sm.wflag[w] = f;
        sm.wseg[w] = v;
    }
    const int pos = seq_block_excl_int(ns, sm, nullptr);  // synchronises: wflag / wseg visible
    bool fc = false;
    Seg vc = sm.open;
    for (int q = 0; q < w; ++q) {
        bool fq = sm.wflag[q];
        Seg vq = sm.wseg[q];
        seq::seg_op(fc, vc, fq, vq);
        fc = fq;
        vc = vq;
    }
    seq::seg_op(fc, vc, fe, ve);  // ve: the segment open before this thread's first element
    // pass B: emit the segment that each start closes
    Seg open = ve;
    pb = prevB0;
    int k = sm.items + pos;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        if (bj[j] == kSeqPadB) break;
        const Seg vj = value(j);
        if (bj[j] != pb || bj[j] == kSeqRawB) {
            if (k < cap) items[k] = seq::Item{open.kind, open.B, open.d.d0, open.d.d1, open.start, base + e0 + j - open.start};
            ++k;
            open = vj;
        } else {
            open = seq::seg_combine(open, vj);
        }
        pb = bj[j];
    }
    __syncthreads();  // every thread has read sm.open / sm.items
    if (threadIdx.x == kSolveThreads - 1) {
        sm.open = open;
        sm.open_B = bj[EPT - 1];
        sm.items = k;
    }
    __syncthreads();
}

// Thread 0: append a run of binade bt starting at `base` to the CTA's open segment (or close
// the open segment into the list and start a new one).
__device__ __forceinline__ void seq_merge_run(SeqSmem& sm, int bt, const seq::Pair& t, int64_t base, seq::Item* items,
                                              int cap) {
    seq::Seg& o = sm.open;
    if (o.kind == seq::kRun && o.B == bt && sm.open_B == bt) {
        o.d = seq::pcompose(o.d, t);
    } else {
        if (o.kind != seq::kEmpty) {
            if (sm.items < cap) items[sm.items] = seq::Item{o.kind, o.B, o.d.d0, o.d.d1, o.start, base - o.start};
            ++sm.items;
        }
        o = seq::Seg{seq::kRun, bt, t, base};
    }
    sm.open_B = bt;
}

// Fast tile (the whole tile predicted in binade bt): the ordered summary of this thread's
// elements x (already |.|, zeros past the end), reduced over the block in element order and
// merged into the CTA's open segment by thread 0.  One block barrier; the warp summaries are
// double-buffered by `buf` so consecutive fast tiles need no second one.
template <int EPT>
__device__ __forceinline__ void seq_fast_tile(SeqSmem& sm, const double (&x)[EPT], int bt, int64_t base,
                                              seq::Item* items, int cap, int buf) {
    using seq::Seg;
    // Without rounding ties the increment does not depend on the parity: a plain integer sum.
    {
        bool tie = false, big = false;
        uint64_t r = 0;
#pragma unroll
        for (int j = 0; j < EPT; ++j) r += seq::elem_r0(x[j], bt, tie, big);
        if (!__syncthreads_or(tie || big)) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);  // <= 32 * 8 * 2^53
            if ((threadIdx.x & 31) == 0) sm.wpair[buf][threadIdx.x >> 5] = seq::Pair{r, r};
            __syncthreads();
            if (threadIdx.x == 0) {
                uint64_t t = 0;
                for (int q = 0; q < kSolveThreads / 32; ++q) t = seq::sat_add(t, sm.wpair[buf][q].d0);
                seq_merge_run(sm, bt, seq::Pair{t, t}, base, items, cap);
            }
            return;
        }
    }
    seq::Pair d{0, 0};
#pragma unroll
    for (int j = 0; j < EPT; ++j) d = seq::pcompose(d, seq::elem_pair(x[j], bt));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // ordered: lane l absorbs lane l + o
        const uint64_t q0 = __shfl_down_sync(0xffffffffu, d.d0, o);
        const uint64_t q1 = __shfl_down_sync(0xffffffffu, d.d1, o);
        if ((lane & (2 * o - 1)) == 0) d = seq::pcompose(d, seq::Pair{q0, q1});
    }
    if (lane == 0) sm.wpair[buf][w] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        seq::Pair t{0, 0};
        for (int q = 0; q < kSolveThreads / 32; ++q) t = seq::pcompose(t, sm.wpair[buf][q]);
        seq_merge_run(sm, bt, t, base, items, cap);
    }
}

// Close the range's open segment at global index end (thread 0); returns the item count.
__device__ __forceinline__ int seq_close(SeqSmem& sm, int64_t end, seq::Item* items, int cap) {
    int k = sm.items;
    const seq::Seg& o = sm.open;
    if (o.kind != seq::kEmpty) {
        if (k < cap) items[k] = seq::Item{o.kind, o.B, o.d.d0, o.d.d1, o.start, end - o.start};
        ++k;
    }
    return k;
}

// One item on the integer state: a run in the current binade is m += d[m & 1] (renormalised
// when it lands exactly on 2^(B+1)); anything else goes through the double value.  Returns
// false when the state became non-finite (the sum overflowed: it stays inf).
template <class Walk>
__device__ __forceinline__ bool seq_step(SeqState& st, int kind, int B, uint64_t d0, uint64_t d1, int64_t start,
                                         int64_t len, Walk walk) {
    if (kind == seq::kRun && B == st.B) {
        const uint64_t mm = st.m + ((st.m & 1) ? d1 : d0);
        if (mm < seq::kTwo53) {
            st.m = mm;
            return true;
        }
        if (mm == seq::kTwo53) {
            if (st.B + 1 > 1023) return false;
            st.B += 1;
            st.m = seq::kTwo52;
            return true;
        }
    }
    if (kind == seq::kEmpty) return true;
    double s = st.value();
    if (kind == seq::kRaw) s = __dadd_rn(s, __longlong_as_double(static_cast<long long>(d0)));
    else s = walk(s, start, start + len);
    if (!isfinite(s)) return false;
    st.set(s);
    return true;
}

// One item of the walk: acc <- acc + item; walk(acc, lo, hi) adds elements [lo, hi) one by
// one (the reference's loop) when the item is raw-range / mixed or its run check fails.
template <class Walk>
__device__ __forceinline__ void seq_apply_item(double& acc, const seq::Item& it, Walk walk) {
    if (it.kind == seq::kEmpty) return;
    if (it.kind == seq::kRaw) {
        acc = __dadd_rn(acc, __longlong_as_double(static_cast<long long>(it.d0)));
        return;
    }
    if (it.kind == seq::kRun && seq::apply_run(acc, it.B, seq::Pair{it.d0, it.d1})) return;
    acc = walk(acc, it.start, it.start + it.len);
}

// One item on the state s (as its bits), carefully: a run in s's binade as an integer add
// (checked), a raw element as __dadd_rn, anything else the reference's loop over its elements.
// False: the sum overflowed (it stays inf).
template <class Walk>
__device__ __noinline__ bool seq_item_slow(uint64_t& bits, int kind, int B, uint64_t d0, uint64_t d1, longlong2 r,
                                           Walk walk, bool debug) {
    if (kind == seq::kEmpty) return true;
    double s = __longlong_as_double(static_cast<long long>(bits));
    if (kind == seq::kRaw) {
        s = __dadd_rn(s, __longlong_as_double(static_cast<long long>(d0)));
    } else if (kind != seq::kRun || !seq::apply_run(s, B, seq::Pair{d0, d1})) {
        if (debug) printf("seqsum walk: kind %d B %d start %lld len %lld\n", kind, B, r.x, r.y);
        s = walk(s, r.x, r.x + r.y);
    }
    bits = static_cast<uint64_t>(__double_as_longlong(s));
    return isfinite(s);
}

// The composer's inner loop over m staged items (thread 0), on the bits of s.  Within a binade
// the bits of s are ((B + 1022) << 52) + m for every B (subnormals included), and 2^(B+1)'s
// bits are what m = 2^53 gives -- so a run is bits += d[bits & 1] and a raw element one
// __dadd_rn: a chain of about three dependent instructions per item.  Whether each run really
// started in its binade and stayed in it (lo <= bits, result <= hi) is checked off the chain;
// a batch with any failure is redone item by item with seq_item_slow.
constexpr int kSeqWalkU = 8;
template <class Walk>
__device__ __noinline__ bool seq_walk_batch(uint64_t& io, const int* kind, const int* bb, const uint64_t* d0,
                                            const uint64_t* d1, const uint64_t* lo, const uint64_t* hi,
                                            const longlong2* pos, int m, Walk walk, bool debug) {
    // staged so that the chain has no branches: empties (and the padding up to a multiple of
    // kSeqWalkU) are zero runs valid anywhere, mixed items have lo > hi (always "bad"), a raw
    // item has lo = 0, hi = ~0 and its value in d0
    uint64_t bits = io;
    for (int q0 = 0; q0 < m; q0 += kSeqWalkU) {
        const uint64_t start = bits;
        uint64_t a0[kSeqWalkU], a1[kSeqWalkU], l[kSeqWalkU], h[kSeqWalkU];
        bool raw[kSeqWalkU];
#pragma unroll
        for (int u = 0; u < kSeqWalkU; ++u) {
            a0[u] = d0[q0 + u];
            a1[u] = d1[q0 + u];
            l[u] = lo[q0 + u];
            h[u] = hi[q0 + u];
            raw[u] = kind[q0 + u] == seq::kRaw;
        }
        unsigned bad = 0;
#pragma unroll
        for (int u = 0; u < kSeqWalkU; ++u) {
            const uint64_t odd = 0ull - (bits & 1ull);
            const uint64_t run = bits + (a0[u] ^ ((a0[u] ^ a1[u]) & odd));
            const uint64_t rw = static_cast<uint64_t>(__double_as_longlong(
                __dadd_rn(__longlong_as_double(static_cast<long long>(bits)), __longlong_as_double(static_cast<long long>(a0[u])))));
            bad |= static_cast<unsigned>(bits < l[u]) | static_cast<unsigned>(run > h[u]);
            bits = raw[u] ? rw : run;
        }
        if (bad | static_cast<unsigned>(bits >= 0x7ff0000000000000ull)) {
            if (debug) printf("seqsum walk: slow batch at %d\n", q0);
            bits = start;
            for (int q = q0; q < min(m, q0 + kSeqWalkU); ++q)
                if (!seq_item_slow(bits, kind[q], bb[q], d0[q], d1[q], pos[q], walk, debug)) return false;
        }
    }
    io = bits;
    return true;
}

// Stage one item for seq_walk_batch: a run of binade B must start in [2^B, 2^(B+1)) (B = -1022:
// from 0) and end <= 2^(B+1); raw items and empties are valid anywhere (empties are zero runs);
// mixed items (or a run with an impossible binade) always fail -> the slow path.
__device__ __forceinline__ void seq_stage(int kind, int B, uint64_t d0, uint64_t d1, uint64_t& o0, uint64_t& o1,
                                          uint64_t& lo, uint64_t& hi) {
    o0 = kind == seq::kEmpty ? 0ull : d0;
    o1 = kind == seq::kEmpty ? 0ull : d1;
    lo = 0ull;
    hi = ~0ull;
    if (kind == seq::kRun) {
        if (B >= -1022 && B <= 1023) {
            lo = B == -1022 ? 0ull : static_cast<uint64_t>(B + 1023) << 52;
            hi = static_cast<uint64_t>(B + 1024) << 52;
        } else {
            lo = ~0ull;
            hi = 0ull;
        }
    } else if (kind == seq::kMixed) {
        lo = ~0ull;
        hi = 0ull;
    }
}
