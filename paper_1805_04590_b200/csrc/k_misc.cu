// k_misc.cu -- K1 (guide derivative) and K6 (solve prologue) for sm_100a.
#include "dts_device.cuh"
#include "dts_launch.h"

namespace dts {

// K1: domain-transform increments between adjacent pixels (Eqs. 8-9 with
// the square restored, R1; sigma scaling R2):
//     d_x[r][c] = sqrt(1 + (sigma_s/sigma_r)^2 sum_k (I[r][c][k] - I[r][c-1][k])^2), d_x[r][0] = +inf
//     d_y[r][c] likewise with row r-1, d_y[0][c] = +inf; columns c >= W (pitch padding) = +inf.
// One thread per pixel; a warp reads 32 consecutive HWC pixels (one contiguous
// 32*C-float span) of rows r and r-1; the left neighbour comes from the lane to the
// left (shuffle) so the guide is streamed once (row r-1 is re-read from L2).
template <int CMAX>
__global__ void __launch_bounds__(256) k_guide_deriv(const float* __restrict__ guide, int C, float ratio2,
                                                     Geometry g, float* __restrict__ dx, float* __restrict__ dy) {
    const int64_t r = blockIdx.y;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.pitch) return;
    const int lane = threadIdx.x & 31;
    float sx = 0.f, sy = 0.f;
    const bool in = c < g.W;
    const float* pr = guide + (r * g.W + c) * C;
    const float* pl = pr - C;
    const float* pu = pr - g.W * C;
    for (int k = 0; k < C; ++k) {
        const float v = in ? __ldg(pr + k) : 0.f;
        // left neighbour's channel k: from lane-1, or a load for lane 0
        float left = __shfl_up_sync(FULL, v, 1);
        if (lane == 0 && in && c > 0) left = __ldg(pl + k);
        const float up = (in && r > 0) ? __ldg(pu + k) : 0.f;
        const float ex = v - left, ey = v - up;
        sx = fmaf(ex, ex, sx);
        sy = fmaf(ey, ey, sy);
    }
    const int64_t o = r * g.pitch + c;
    dx[o] = (in && c > 0) ? sqrtf(fmaf(ratio2, sx, 1.f)) : __int_as_float(0x7f800000);
    dy[o] = (in && r > 0) ? sqrtf(fmaf(ratio2, sy, 1.f)) : __int_as_float(0x7f800000);
}

cudaError_t launch_guide_deriv(const float* guide, int C, float ratio2, const Geometry& g, float* dx, float* dy,
                               cudaStream_t s) {
    dim3 block(256);
    dim3 grid((unsigned)((g.pitch + 255) / 256), (unsigned)g.H);
    k_guide_deriv<0><<<grid, block, 0, s>>>(guide, C, ratio2, g, dx, dy);
    return cudaGetLastError();
}

// K6: planar state from the HWC target, chat = c / S (R7).
__global__ void __launch_bounds__(256) k_prologue(const float* __restrict__ target, const float* __restrict__ conf,
                                                  int Ct, Geometry g, const float* __restrict__ S, int support_mode,
                                                  float* __restrict__ Z, float* __restrict__ T,
                                                  float* __restrict__ chat) {
    const int64_t r = blockIdx.y;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.W) return;
    const int64_t p = r * g.W + c;
    const int64_t o = r * g.pitch + c;
    for (int v = 0; v < Ct; ++v) {
        const float t = __ldg(target + p * Ct + v);
        Z[v * g.plane + o] = t;
        T[v * g.plane + o] = t;
    }
    const float cv = __ldg(conf + p);
    chat[o] = support_mode == 1 ? cv : cv / S[o];
}

cudaError_t launch_prologue(const float* target, const float* conf, int Ct, const Geometry& g, const float* S,
                            int support_mode, float* Z, float* T, float* chat, cudaStream_t s) {
    dim3 block(256);
    dim3 grid((unsigned)((g.W + 255) / 256), (unsigned)g.H);
    k_prologue<<<grid, block, 0, s>>>(target, conf, Ct, g, S, support_mode, Z, T, chat);
    return cudaGetLastError();
}

// opt-in input validation: counters[0] = non-finite target/confidence values,
// counters[1] = confidences outside [0, 1]
__global__ void k_check_inputs(const float* __restrict__ target, const float* __restrict__ conf, int Ct, int64_t n,
                               unsigned int* counters) {
    unsigned int bad = 0, range = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float cv = conf[i];
        if (!isfinite(cv)) ++bad;
        else if (cv < 0.f || cv > 1.f) ++range;
        for (int v = 0; v < Ct; ++v)
            if (!isfinite(target[i * Ct + v])) ++bad;
    }
    bad = __reduce_add_sync(FULL, bad);
    range = __reduce_add_sync(FULL, range);
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicAdd(&counters[0], bad);
        if (range) atomicAdd(&counters[1], range);
    }
}

cudaError_t launch_check_inputs(const float* target, const float* conf, int Ct, int64_t H, int64_t W,
                                unsigned int* counters, cudaStream_t s) {
    k_check_inputs<<<296, 256, 0, s>>>(target, conf, Ct, H * W, counters);
    return cudaGetLastError();
}

}  // namespace dts
