// gs_device.cuh -- device-side building blocks of the exponential-Euler hot path.
//
// Arithmetic contract: every floating-point operation on the parity
// path is an explicit IEEE round-to-nearest double op (__dmul_rn / __dadd_rn), in the
// reference's order, and the library is compiled with -fmad=false, so no FMA
// contraction can change a bit relative to the reference's x86-64 (no-FMA) build.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gs {

constexpr int kTX = 32;                 // tile width in x  (one warp = one coalesced x-row)
constexpr int kTY = 8;                  // tile height in y (8 warps)
constexpr int kThreads = kTX * kTY;     // 256 threads per CTA
constexpr int kMaxDegree = 55;          // kMaxTaylorDegree (expact.hpp:39)
constexpr int kMaxLoggedStages = 256;

// ---------------------------------------------------------------------------------
// Operator description: the matrix-free form of assemble_diffusion (stencil.cpp:5-43)
// ---------------------------------------------------------------------------------
struct StencilOp {
    int nx, ny, nz;
    int64_t n, sy, sz;
    const uint8_t* pal;   // palette index per voxel (palette mode), or nullptr
    const double* dvox;   // per-voxel D (fp64 mode, > 256 distinct values), or nullptr
    const double* wtab;   // [256] w_k = D_k * (1/(h*h)), computed on the host like stencil.cpp:8,23
    double inv_h2;        // 1.0 / (h*h)   (stencil.cpp:8)
    // work decomposition: tiles of kTX x kTY columns, z-chunks of zc planes
    int tiles_x, tiles_y, zc, chunks_z;
    int64_t n_items;
    // generic operator (SparseOperator, sparse.hpp:13-38): CSR with sorted unique columns.
    // Non-null -> every sweep applies this matrix instead of the stencil.
    const int64_t* csr_offs;
    const int32_t* csr_cols;
    const double* csr_vals;
};

// Row r of a generic CSR operator applied to x exactly as SparseOperator::apply does
// (sparse.cpp:54-58): acc = 0; acc += val*x[col] in storage order.
__device__ __forceinline__ double csr_row_apply(const StencilOp& op, int64_t r, const double* x) {
    double acc = 0.0;
    for (int64_t q = op.csr_offs[r]; q < op.csr_offs[r + 1]; ++q)
        acc = __dadd_rn(acc, __dmul_rn(op.csr_vals[q], x[op.csr_cols[q]]));
    return acc;
}

// Per-voxel row coefficients: w = D_v / h^2 and whether the row exists (D_v != 0).
struct RowCoef {
    double w;
    bool live;
};

__device__ __forceinline__ RowCoef row_coef(const StencilOp& op, const double* s_wtab, int64_t v) {
    RowCoef r;
    if (op.pal) {
        r.w = s_wtab[op.pal[v]];
        // D_k != 0  <=>  the stored w_k != 0 unless D_k*inv_h2 underflowed; the host
        // rejects that case, so w != 0 is the stencil.cpp:22 test.
        r.live = r.w != 0.0;
    } else {
        const double d = op.dvox[v];
        r.w = __dmul_rn(d, op.inv_h2);
        r.live = d != 0.0;
    }
    return r;
}

// Row v of the operator applied to x, accumulated exactly as SparseOperator::apply does
// (sparse.cpp:54-58) over the sorted row of assemble_diffusion: columns v-sz, v-sy, v-1,
// v, v+1, v+sy, v+sz; off-diagonals w, diagonal (-cnt)*w (stencil.cpp:30-36).  Missing
// neighbours are passed as 0.0: w*0 adds a signed zero to an accumulator that can never
// be -0 (it starts at +0.0), so the sum is bit-identical to skipping the entry.
__device__ __forceinline__ double row_apply(const RowCoef& c, int cnt, double xzm, double xym, double xxm,
                                            double xc, double xxp, double xyp, double xzp) {
    const double diag = __dmul_rn(static_cast<double>(-cnt), c.w);
    double acc = __dadd_rn(0.0, __dmul_rn(c.w, xzm));
    acc = __dadd_rn(acc, __dmul_rn(c.w, xym));
    acc = __dadd_rn(acc, __dmul_rn(c.w, xxm));
    acc = __dadd_rn(acc, __dmul_rn(diag, xc));
    acc = __dadd_rn(acc, __dmul_rn(c.w, xxp));
    acc = __dadd_rn(acc, __dmul_rn(c.w, xyp));
    acc = __dadd_rn(acc, __dmul_rn(c.w, xzp));
    return c.live ? acc : 0.0;   // empty row (stencil.cpp:22)
}

// Same row with the diagonal's (double)(-cnt) precomputed by the caller (exact small integer).
__device__ __forceinline__ double row_apply_nc(double w, bool live, double negcnt, double xzm, double xym, double xxm,
                                               double xc, double xxp, double xyp, double xzp) {
    const double diag = __dmul_rn(negcnt, w);
    double acc = __dadd_rn(0.0, __dmul_rn(w, xzm));
    acc = __dadd_rn(acc, __dmul_rn(w, xym));
    acc = __dadd_rn(acc, __dmul_rn(w, xxm));
    acc = __dadd_rn(acc, __dmul_rn(diag, xc));
    acc = __dadd_rn(acc, __dmul_rn(w, xxp));
    acc = __dadd_rn(acc, __dmul_rn(w, xyp));
    acc = __dadd_rn(acc, __dmul_rn(w, xzp));
    return live ? acc : 0.0;
}

// The same without the dead-row select, for sweeps whose results are checked: with w = 0 and
// finite inputs every product is a signed zero and the sum is +0.0, the select's value; only
// a non-finite neighbour makes a dead row non-finite (0 * inf), and a sweep whose bounding
// maxima see a non-finite value is rerun with the selects (sweep2_tma<.., kExact = true>).
__device__ __forceinline__ double row_apply_ns(double w, double negcnt, double xzm, double xym, double xxm, double xc,
                                               double xxp, double xyp, double xzp) {
    const double diag = __dmul_rn(negcnt, w);
    double acc = __dadd_rn(0.0, __dmul_rn(w, xzm));
    acc = __dadd_rn(acc, __dmul_rn(w, xym));
    acc = __dadd_rn(acc, __dmul_rn(w, xxm));
    acc = __dadd_rn(acc, __dmul_rn(diag, xc));
    acc = __dadd_rn(acc, __dmul_rn(w, xxp));
    acc = __dadd_rn(acc, __dmul_rn(w, xyp));
    acc = __dadd_rn(acc, __dmul_rn(w, xzp));
    return acc;
}

// ---------------------------------------------------------------------------------
// Order-free reductions
// ---------------------------------------------------------------------------------
// |x| maxima are accumulated as the IEEE bit pattern of a non-negative double, which
// orders like the value; NaN is dropped exactly as std::max(m, |x|) drops it
// (expact.cpp:15-19), so the result equals the reference's serial max bit for bit.
__device__ __forceinline__ double nan_dropping_max(double m, double x) { return (m < x) ? x : m; }

// |x| by clearing the sign bit in the integer pipe (fabs would cost an fp64 DADD with an
// |.| modifier); identical to fabs for every input, NaN included.
__device__ __forceinline__ double abs_bits(double x) {
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}
__device__ __forceinline__ double max_abs(double m, double x) { return nan_dropping_max(m, abs_bits(x)); }

// Bounding maxima.  The high word of |x| without its sign, as an unsigned key (exponent and
// 20 mantissa bits), orders like |x| up to the discarded low word: max over keys costs two
// integer instructions per value instead of the DSETP/FSEL max of the exact path.  From the
// maximum key K, key_lower(K) <= max|x| <= key_upper(key_lower(K)) for finite values; a key
// of an inf or NaN (K >= 0xffe00000) maps to +inf, which callers treat as "bounds unknown".
__device__ __forceinline__ unsigned max_key(double x) { return static_cast<unsigned>(__double2hiint(x)) << 1; }
__device__ __forceinline__ double key_lower(unsigned k) {
    return __hiloint2double(static_cast<int>(min(k, 0xffe00000u) >> 1), 0);
}
__device__ __forceinline__ double key_upper(double lower) {
    return __hiloint2double(__double2hiint(lower), static_cast<int>(0xffffffffu));
}

// Signed doubles mapped to an unsigned order-preserving key (for min/max of u).
__device__ __forceinline__ unsigned long long ordered_key(double x) {
    unsigned long long b = __double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered_key(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(b);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = nan_dropping_max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Fixed-shape tree: deterministic for a fixed launch geometry.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace gs
