// gs_vtkfmt.cu -- the VTK value column formatted on the GPU (snapshots of resident states).
//
// write_vtk prints every value with snprintf("%.17g") (vtk.cpp:16-20, :81).  For a snapshot
// of the resident state the values are already in HBM, so the text is made there:
//   1. len_kernel: each thread formats its value with the exact %.17g algorithm of
//      gsio::fmt17 (128-bit powers of ten, from the same table) and stores the length;
//      values within 2 ulp of a rounding tie are flagged (the host formatter's libc case);
//   2. an exclusive scan of the lengths (CUB) gives every value's byte offset;
//   3. write_kernel formats again and stores the text at its offset.
// The host copies the text back (D2H on the snapshot stream) and writes it.  A flagged
// value (never seen in practice) makes the caller fall back to the host formatter, so the
// bytes always equal the reference's.
#include <cub/cub.cuh>

#include <algorithm>

#include "gs_io.hpp"
#include "gs_vtkfmt.cuh"

namespace gs {

namespace {

__constant__ unsigned long long c_p10_hi[gsio::kPow10Count];
__constant__ unsigned long long c_p10_lo[gsio::kPow10Count];
__constant__ int c_p10_b[gsio::kPow10Count];
__constant__ int c_p10_qmin;

__device__ __forceinline__ int put(char* o, const char* s) {
    int k = 0;
    while (s[k]) {
        o[k] = s[k];
        ++k;
    }
    return k;
}

// Exactly printf("%.17g", v) for every double (see gsio::fmt17); *tie set when the rounding
// decision is within the table's error of a tie (the caller must not trust the text then).
__device__ int fmt17_dev(double v, char* out, bool* tie) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    const int bexp = static_cast<int>((bits >> 52) & 0x7ff);
    const unsigned long long frac = bits & ((1ull << 52) - 1);
    const bool neg = bits >> 63;
    char* o = out;
    if (bexp == 0x7ff) {  // glibc: inf / -inf / nan / -nan
        if (neg) *o++ = '-';
        return static_cast<int>(o - out) + put(o, frac ? "nan" : "inf");
    }
    if (bexp == 0 && frac == 0) {
        if (neg) *o++ = '-';
        *o++ = '0';
        return static_cast<int>(o - out);
    }
    unsigned long long M;
    int e;
    if (bexp == 0) {
        const int lz = __clzll(static_cast<long long>(frac));
        M = frac << lz;
        e = -1074 - lz;
    } else {
        M = (frac | (1ull << 52)) << 11;
        e = bexp - 1075 - 11;
    }
    const int x = e + 63;
    int e10 = (x * 78913) >> 18;
    unsigned long long N = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const int qi = 16 - e10 - c_p10_qmin;
        const unsigned long long Fhi = c_p10_hi[qi], Flo = c_p10_lo[qi];
        // P = M * (Fhi:Flo) as w2:w1:w0
        const unsigned long long ll = M * Flo, lh = __umul64hi(M, Flo);
        const unsigned long long hl = M * Fhi, hh = __umul64hi(M, Fhi);
        const unsigned long long w1 = lh + hl;
        const unsigned long long w2 = hh + (w1 < lh ? 1ull : 0ull);
        (void)ll;
        const int sh = -(e + c_p10_b[qi]);
        const int r = sh - 128;
        if (r < 1 || r > 63) {
            *tie = true;
            return 0;
        }
        const unsigned long long I = w2 >> r;
        if (I >= 100000000000000000ull && attempt == 0) {
            ++e10;
            continue;
        }
        // fraction (w2 mod 2^r):w1 against half = 2^(r-1):0, with a margin of 2 in the low limb
        const unsigned long long fh = w2 & ((1ull << r) - 1), fl = w1;
        const unsigned long long hh2 = 1ull << (r - 1);
        // fhi + 2 < half ?
        const unsigned long long fl2 = fl + 2;
        const unsigned long long fh2 = fh + (fl2 < fl ? 1ull : 0ull);
        if (fh2 < hh2) {
            N = I;
        } else if (fh > hh2 || (fh == hh2 && fl > 0)) {
            N = I + 1;
        } else {
            *tie = true;
            return 0;
        }
        break;
    }
    if (N >= 100000000000000000ull) {
        N /= 10;
        ++e10;
    }
    if (N < 10000000000000000ull) {
        *tie = true;
        return 0;
    }
    char dig[17];
    for (int i = 16; i >= 0; --i) {
        dig[i] = static_cast<char>('0' + N % 10);
        N /= 10;
    }
    int nd = 17;
    while (nd > 1 && dig[nd - 1] == '0') --nd;
    if (neg) *o++ = '-';
    const int X = e10;
    if (X < -4 || X >= 17) {
        *o++ = dig[0];
        if (nd > 1) {
            *o++ = '.';
            for (int i = 1; i < nd; ++i) *o++ = dig[i];
        }
        *o++ = 'e';
        int ax = X;
        if (ax < 0) {
            *o++ = '-';
            ax = -ax;
        } else {
            *o++ = '+';
        }
        if (ax >= 100) {
            *o++ = static_cast<char>('0' + ax / 100);
            ax %= 100;
        }
        *o++ = static_cast<char>('0' + ax / 10);
        *o++ = static_cast<char>('0' + ax % 10);
    } else if (X >= 0) {
        for (int i = 0; i <= X; ++i) *o++ = dig[i];
        if (nd > X + 1) {
            *o++ = '.';
            for (int i = X + 1; i < nd; ++i) *o++ = dig[i];
        }
    } else {
        *o++ = '0';
        *o++ = '.';
        for (int i = 0; i < -X - 1; ++i) *o++ = '0';
        for (int i = 0; i < nd; ++i) *o++ = dig[i];
    }
    return static_cast<int>(o - out);
}

__global__ void len_kernel(const double* __restrict__ u, int64_t n, unsigned long long* __restrict__ lens,
                           int* __restrict__ tie_flag) {
    char buf[32];
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        bool tie = false;
        const int l = fmt17_dev(u[i], buf, &tie);
        if (tie) atomicExch(tie_flag, 1);
        lens[i] = static_cast<unsigned long long>(l + 1);  // + '\n'
    }
}

__global__ void write_kernel(const double* __restrict__ u, int64_t n, const unsigned long long* __restrict__ offs,
                             char* __restrict__ text) {
    char buf[32];
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        bool tie = false;
        const int l = fmt17_dev(u[i], buf, &tie);
        char* o = text + offs[i];
        for (int k = 0; k < l; ++k) o[k] = buf[k];
        o[l] = '\n';
    }
}

// material codes 0..9 as "d\n" (vtk.cpp:85); the caller checks that every code is < 10
__global__ void labels_kernel(const uint8_t* __restrict__ lab, int64_t n, char* __restrict__ text) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        text[2 * i] = static_cast<char>('0' + lab[i]);
        text[2 * i + 1] = '\n';
    }
}

}  // namespace

cudaError_t vtkfmt_init() {
    static bool done = false;
    if (done) return cudaSuccess;
    static uint64_t hi[gsio::kPow10Count], lo[gsio::kPow10Count];
    static int b[gsio::kPow10Count];
    int qmin = 0, count = 0;
    gsio::pow10_table_export(hi, lo, b, &qmin, &count);
    cudaError_t e = cudaMemcpyToSymbol(c_p10_hi, hi, sizeof hi);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_p10_lo, lo, sizeof lo);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_p10_b, b, sizeof b);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_p10_qmin, &qmin, sizeof qmin);
    done = e == cudaSuccess;
    return e;
}

size_t vtkfmt_scratch_bytes(int64_t n) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, static_cast<unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<int>(n));
    return tmp;
}

cudaError_t vtkfmt_values(const double* u, int64_t n, VtkfmtScratch& s, cudaStream_t stream) {
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
    cudaError_t e = cudaMemsetAsync(s.tie, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    len_kernel<<<blocks, 256, 0, stream>>>(u, n, s.lens, s.tie);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    size_t tmp = s.scan_bytes;
    e = cub::DeviceScan::ExclusiveSum(s.scan_tmp, tmp, s.lens, s.offs, static_cast<int>(n), stream);
    if (e != cudaSuccess) return e;
    // total = offs[n-1] + lens[n-1], fetched by the host with the text
    write_kernel<<<blocks, 256, 0, stream>>>(u, n, s.offs, s.text);
    return cudaGetLastError();
}

cudaError_t vtkfmt_labels(const uint8_t* lab, int64_t n, char* text, cudaStream_t stream) {
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
    labels_kernel<<<blocks, 256, 0, stream>>>(lab, n, text);
    return cudaGetLastError();
}

}  // namespace gs
