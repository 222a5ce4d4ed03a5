// tma_probe2.cu -- parametric tensor-TMA probe (debug tool).
//   ./tma_probe2 RANK DTYPE(0=f64,1=f32,2=u8) N0 N1 N2 B0 B1 B2 [swizzle] [l2promo] [oob]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gs_tma.cuh"

using namespace gs;

struct P {
    CUtensorMap map;
    unsigned char* out;
    int rank;
    unsigned bytes;
    int c0, c1, c2;
};

__global__ void k(const __grid_constant__ P p) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, p.bytes);
        uint64_t m = reinterpret_cast<uint64_t>(&p.map);
        if (p.rank == 1)
            asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                         ::"r"(smem_u32(sm)), "l"(m), "r"(p.c0), "r"(smem_u32(&bar)) : "memory");
        else if (p.rank == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(sm)), "l"(m), "r"(p.c0), "r"(p.c1), "r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(sm)), "l"(m), "r"(p.c0), "r"(p.c1), "r"(p.c2), "r"(smem_u32(&bar)) : "memory");
    }
    mbar_wait(&bar, 0);
    for (unsigned i = threadIdx.x; i < p.bytes; i += blockDim.x) p.out[i] = sm[i];
}

int main(int argc, char** argv) {
    int rank = atoi(argv[1]), dt = atoi(argv[2]);
    cuuint64_t dims[3] = {(cuuint64_t)atoll(argv[3]), (cuuint64_t)atoll(argv[4]), (cuuint64_t)atoll(argv[5])};
    cuuint32_t box[3] = {(cuuint32_t)atoi(argv[6]), (cuuint32_t)atoi(argv[7]), (cuuint32_t)atoi(argv[8])};
    int swz = argc > 9 ? atoi(argv[9]) : 0, l2 = argc > 10 ? atoi(argv[10]) : 0, oob = argc > 11 ? atoi(argv[11]) : 0;
    int es = dt == 0 ? 8 : dt == 1 ? 4 : 1;
    CUtensorMapDataType t = dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                            : dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    size_t n = dims[0] * (rank > 1 ? dims[1] : 1) * (rank > 2 ? dims[2] : 1);
    void* d;
    cudaMalloc(&d, n * es);
    cudaMemset(d, 1, n * es);
    cuuint64_t st[2] = {dims[0] * es, dims[0] * dims[1] * es};
    cuuint32_t estr[3] = {1, 1, 1};
    P p{};
    CUresult r = cuTensorMapEncodeTiled(&p.map, t, rank, d, dims, st, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        (CUtensorMapSwizzle)swz, (CUtensorMapL2promotion)l2,
                                        (CUtensorMapFloatOOBfill)oob);
    p.rank = rank;
    p.c0 = argc > 12 ? atoi(argv[12]) : 0;
    p.c1 = argc > 13 ? atoi(argv[13]) : 0;
    p.c2 = argc > 14 ? atoi(argv[14]) : 0;
    p.bytes = box[0] * (rank > 1 ? box[1] : 1) * (rank > 2 ? box[2] : 1) * es;
    cudaMalloc(&p.out, p.bytes);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k<<<1, 128, p.bytes + 1024>>>(p);
    cudaError_t e = cudaDeviceSynchronize();
    printf("coords %d %d %d rank %d dt %d dims %llu %llu %llu box %u %u %u swz %d l2 %d: encode %d -> %s\n", p.c0, p.c1, p.c2, rank, dt,
           (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2], box[0], box[1], box[2],
           swz, l2, (int)r, cudaGetErrorString(e));
    return e != cudaSuccess;
}
