// tma_probe.cu -- isolate TMA / mbarrier PTX forms on the B200 (debug tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_2402_02273_b200/csrc -o tma_probe tma_probe.cu
//   ./tma_probe VARIANT NX NY NZ
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gs_tma.cuh"

using namespace gs;

struct Params {
    CUtensorMap map;
    const CUtensorMap* gmap;
    const double* src;
    CUtensorMap lmap;
    double* out;
    unsigned char* lout;
    int variant;
    int x0, y0, z;
};

constexpr int BX = 66, BY = 18;

__global__ void probe(const __grid_constant__ Params p) {
    __shared__ __align__(128) double tile[BY * BX + 16];
    __shared__ __align__(128) unsigned char lt[64 * 16];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        if (p.variant >= 1 && p.variant < 10) mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (p.variant >= 2 && p.variant < 10) fence_proxy_async_global();
        if (p.variant >= 3 && p.variant < 10) tma_prefetch_desc(&p.map);
        uint32_t bytes = BY * BX * 8 + ((p.variant >= 4 && p.variant < 10) ? 64 * 16 : 0);
        if (p.variant == 13) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
        } else if (p.variant == 14) {
            mbar_arrive_expect_tx(&bar, 0);
        } else if (p.variant == 16 || p.variant == 17) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(tile)),
                "l"(reinterpret_cast<uint64_t>(&p.map)), "r"(smem_u32(&bar)), "r"(p.x0), "r"(p.y0), "r"(p.z),
                "l"(0x1000000000000000ull)
                : "memory");
        } else if (p.variant == 18) {
            // plain bulk copy (no tensor map): 4096 bytes from out buffer's source
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(4096) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(tile)), "l"(p.src), "r"(4096), "r"(smem_u32(&bar)) : "memory");
        } else if (p.variant == 10) {
            // no TMA: plain arrive completes the phase
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
        } else {
            mbar_arrive_expect_tx(&bar, bytes);
            tma_load_3d(tile, p.variant == 11 ? p.gmap : &p.map, p.x0, p.y0, p.z, &bar);
        }
        if (p.variant >= 4 && p.variant < 10) tma_load_3d(lt, &p.lmap, p.x0 + 1, p.y0 + 1, p.z, &bar);
    }
    if (p.variant == 12) {
        // CUTLASS-style wait
        asm volatile("{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(&bar)), "r"(0));
    } else {
        mbar_wait(&bar, 0);
    }
    for (int i = threadIdx.x; i < BX * BY; i += blockDim.x) p.out[i] = tile[i];
    if (p.variant >= 4 && p.variant < 10)
        for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) p.lout[i] = lt[i];
}

int main(int argc, char** argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    int nx = argc > 2 ? atoi(argv[2]) : 16, ny = argc > 3 ? atoi(argv[3]) : 16, nz = argc > 4 ? atoi(argv[4]) : 16;
    size_t n = (size_t)nx * ny * nz;
    std::vector<double> h(n);
    std::vector<unsigned char> hl(n);
    for (size_t i = 0; i < n; ++i) {
        h[i] = (double)i;
        hl[i] = (unsigned char)(i % 251);
    }
    double* d;
    unsigned char* dl;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&dl, n);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dl, hl.data(), n, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaFree(0);
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
    printf("entry point query %d, fn %p, direct %p\n", (int)q, (void*)encode, (void*)&cuTensorMapEncodeTiled);
    if (variant == 17) encode = &cuTensorMapEncodeTiled;
    Params p{};
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t st[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
    cuuint64_t st1[2] = {(cuuint64_t)nx, (cuuint64_t)nx * ny};
    cuuint32_t box[3] = {BX, BY, 1}, lbox[3] = {64, 16, 1}, es[3] = {1, 1, 1};
    CUresult r = encode(&p.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = encode(&p.lmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dl, dims, st1, lbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d %d\n", (int)r, (int)r2);
    const unsigned long long* md = reinterpret_cast<const unsigned long long*>(&p.map);
    for (int i = 0; i < 16; ++i) printf("%016llx%s", md[i], (i % 4 == 3) ? "\n" : " ");
    double* out;
    unsigned char* lout;
    cudaMalloc(&out, BX * BY * 8);
    cudaMalloc(&lout, 64 * 16);
    p.out = out;
    p.lout = lout;
    p.variant = variant;
    CUtensorMap* gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &p.map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    p.gmap = gm;
    p.src = d;
    p.x0 = -1;
    p.y0 = -1;
    p.z = 1;
    if (variant >= 5 && variant < 10) {
        void* args[] = {&p};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)probe, dim3(4), dim3(128), args, 0, 0);
        printf("coop launch: %s\n", cudaGetErrorString(e));
    } else {
        probe<<<1, 128>>>(p);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<double> ho(BX * BY);
    cudaMemcpy(ho.data(), out, BX * BY * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < BY; ++y)
        for (int x = 0; x < BX; ++x) {
            int gx = x - 1, gy = y - 1, gz = 1;
            double want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz < nz) ? (double)(gx + (size_t)nx * (gy + (size_t)ny * gz)) : 0.0;
            if (ho[y * BX + x] != want) ++bad;
        }
    printf("variant %d: %d mismatches\n", variant, bad);
    return 0;
}
