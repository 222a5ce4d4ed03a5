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

}  // namespace seq

constexpr int kSeqEPT = 8;                          // elements per thread and tile
constexpr int kSeqTile = kSolveThreads * kSeqEPT;   // elements per tile
constexpr int kSeqItemCap = 512;                    // items per CTA list

struct SeqSmem {
    double dred[kSolveThreads / 32];
    int ired[kSolveThreads / 32];
    seq::Seg wseg[kSolveThreads / 32];
    bool wflag[kSolveThreads / 32];
    int lastB[kSolveThreads];      // per thread: binade of its last element (-2000: raw)
    seq::Seg open;                 // the CTA's open segment carried across its tiles
    int open_B;                    // binade of the previous element (-2000: raw / none)
    int items;                     // items emitted so far
    bool last;
    double bcast;
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
template <int EPT, class Load>
__device__ __forceinline__ void seq_tile_items(SeqSmem& sm, Load load, int64_t base, int cnt, double a_tile,
                                               seq::Item* items, int cap) {
    using seq::Seg;
    const int e0 = static_cast<int>(threadIdx.x) * EPT;
    double x[EPT];
    double ts = 0.0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        x[j] = e0 + j < cnt ? fabs(load(e0 + j)) : 0.0;
        ts = __dadd_rn(ts, x[j]);
    }
    const double a0 = __dadd_rn(a_tile, seq_block_excl_sum(ts, sm, nullptr));
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
