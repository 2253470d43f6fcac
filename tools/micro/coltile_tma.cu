// Micro-benchmark: the column pass's data movement without its arithmetic.  One CTA per SM
// streams 32-column x 640-row tiles: TMA boxes (32 x 32 floats) of x and d land in shared
// memory (double-buffered, the next tile in flight), the tile is written back from shared
// memory.  d is row-major (like d_y) or column-tile-major (each 32-column strip
// contiguous), to see whether strided 128-B segments cap the bandwidth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o coltile_tma coltile_tma.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int TW = 32, BR = 32, NB = 20, TR = BR * NB;  // tile: 32 columns x 640 rows

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(
            smem_u32(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
        : "memory");
}

__global__ void __launch_bounds__(640, 1) k(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap td,
                                            float* __restrict__ y, int H, int W, int pitch, int tiled) {
    // like the cluster column kernel: one landing zone (the next tile lands while this one
    // is in registers), registers <- landing zone, refill, stores straight from registers
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar;
    const int ntx = W / TW, nty = (H + TR - 1) / TR, ntiles = ntx * nty;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int tile) {
        const int tcol = tile % ntx, trow = tile / ntx;
        const int c0 = tcol * TW, r0 = trow * TR;
        mbar_expect(&bar, 2 * TR * TW * 4);
        for (int q = 0; q < NB; ++q) {
            tma2(sm + q * BR * TW, &tx, c0, r0 + q * BR, &bar);
            if (tiled) tma3(sm + (TR + q * BR) * TW, &td, 0, r0 + q * BR, tcol, &bar);
            else tma2(sm + (TR + q * BR) * TW, &td, c0, r0 + q * BR, &bar);
        }
    };
    int k = 0;
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x);
    const int c = threadIdx.x & 31, rg = threadIdx.x >> 5;  // 20 warps x 32 rows
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        mbar_wait(&bar, (uint32_t)(k & 1));
        float xv[BR], dv[BR];
#pragma unroll
        for (int j = 0; j < BR; ++j) {
            xv[j] = sm[(rg * BR + j) * TW + c];
            dv[j] = sm[(TR + rg * BR + j) * TW + c];
        }
        __syncthreads();  // landing zone free
        if (threadIdx.x == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x);
        const int tcol = tile % ntx, trow = tile / ntx;
        float* yt = y + (size_t)(trow * TR + rg * BR) * pitch + tcol * TW + c;
#pragma unroll
        for (int j = 0; j < BR; ++j) yt[(size_t)j * pitch] = xv[j] + dv[j];
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
    const int H = 10240, W = 10240, pitch = 10240;
    const size_t n = (size_t)H * pitch;
    float *x, *d, *dt, *y;
    cudaMalloc(&x, n * 4);
    cudaMalloc(&d, n * 4);
    cudaMalloc(&dt, n * 4);
    cudaMalloc(&y, n * 4);
    cudaMemset(x, 0, n * 4);
    cudaMemset(d, 0, n * 4);
    cudaMemset(dt, 0, n * 4);
    auto e = enc();
    CUtensorMap mx, md, mdt;
    cuuint64_t dims2[2] = {(cuuint64_t)pitch, (cuuint64_t)H};
    cuuint64_t str2[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box2[2] = {TW, BR};
    cuuint32_t es2[2] = {1, 1};
    e(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims2, str2, box2, es2, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    e(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims2, str2, box2, es2, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t dims3[3] = {(cuuint64_t)TW, (cuuint64_t)H, (cuuint64_t)(W / TW)};  // [tile][row][32]
    cuuint64_t str3[2] = {(cuuint64_t)TW * 4, (cuuint64_t)TW * H * 4};
    cuuint32_t box3[3] = {TW, BR, 1};
    cuuint32_t es3[3] = {1, 1, 1};
    e(&mdt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dt, dims3, str3, box3, es3, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = 2 * TR * TW * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const double bytes = 12.0 * H * W;
    for (int tiled = 0; tiled < 2; ++tiled)
        for (int grid : {112, 148}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            k<<<grid, 640, smem>>>(mx, tiled ? mdt : md, y, H, W, pitch, tiled);
            cudaEventRecord(e0);
            for (int i = 0; i < 5; ++i) k<<<grid, 640, smem>>>(mx, tiled ? mdt : md, y, H, W, pitch, tiled);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("d %s grid %3d: %.3f ms per pass, %.0f GB/s (%s)\n", tiled ? "tile-major" : "row-major ", grid, ms / 5,
                   bytes / (ms / 5) / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
