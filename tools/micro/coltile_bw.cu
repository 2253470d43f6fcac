// Micro-benchmark: achievable HBM bandwidth of column-tiled streaming (the access pattern
// of a column pass) vs row streaming.  Each CTA owns a tile of TW columns x RB rows and
// copies it (read x, read d, write x) walking the rows; tiles are assigned so that
// concurrently running CTAs cover adjacent tiles of the same row band (ROWMAJOR=1) or
// different row bands of the same column tile (ROWMAJOR=0).
#include <cstdio>
#include <cuda_runtime.h>
template <int TW>
__global__ void k(const float* __restrict__ x, const float* __restrict__ d, float* __restrict__ y, int H, int W,
                  int pitch, int RB, int ntx, int nty, int rowmajor) {
    const int ntiles = ntx * nty;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tx = rowmajor ? tile % ntx : tile / nty;
        const int ty = rowmajor ? tile / ntx : tile % nty;
        const int c0 = tx * TW, r0 = ty * RB;
        const int lanes = TW / 4;  // float4 per lane
        const int rsub = blockDim.x / lanes;
        const int cc = (threadIdx.x % lanes) * 4, rr = threadIdx.x / lanes;
        for (int r = r0 + rr; r < min(r0 + RB, H); r += rsub) {
            const size_t o = (size_t)r * pitch + c0 + cc;
            float4 a = *reinterpret_cast<const float4*>(x + o);
            float4 b = *reinterpret_cast<const float4*>(d + o);
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
            *reinterpret_cast<float4*>(y + o) = a;
        }
    }
}
template <int TW>
float run(const float* x, const float* d, float* y, int H, int W, int pitch, int RB, int rowmajor, int grid) {
    const int ntx = W / TW, nty = (H + RB - 1) / RB;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<TW><<<grid, 512>>>(x, d, y, H, W, pitch, RB, ntx, nty, rowmajor);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k<TW><<<grid, 512>>>(x, d, y, H, W, pitch, RB, ntx, nty, rowmajor);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}
int main() {
    const int H = 10000, W = 10240, pitch = 10240;
    size_t n = (size_t)H * pitch;
    float *x, *d, *y;
    cudaMalloc(&x, n * 4); cudaMalloc(&d, n * 4); cudaMalloc(&y, n * 4);
    cudaMemset(x, 0, n * 4); cudaMemset(d, 0, n * 4);
    const double bytes = 12.0 * H * W;
    int grids[] = {148, 296, 592, 1184};
    for (int rm = 0; rm < 2; ++rm)
        for (int RB : {64, 128, 640, 10000})
            for (int grid : grids) {
                float t16 = run<16>(x, d, y, H, W, pitch, RB, rm, grid);
                float t32 = run<32>(x, d, y, H, W, pitch, RB, rm, grid);
                float t64 = run<64>(x, d, y, H, W, pitch, RB, rm, grid);
                float t128 = run<128>(x, d, y, H, W, pitch, RB, rm, grid);
                float t256 = run<256>(x, d, y, H, W, pitch, RB, rm, grid);
                printf("rowmajor %d RB %5d grid %4d  GB/s: TW16 %6.0f TW32 %6.0f TW64 %6.0f TW128 %6.0f TW256 %6.0f\n", rm,
                       RB, grid, bytes / t16 / 1e6, bytes / t32 / 1e6, bytes / t64 / 1e6, bytes / t128 / 1e6,
                       bytes / t256 / 1e6);
            }
    return 0;
}
