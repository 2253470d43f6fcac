// k_box.cu -- box (normalised-convolution) variant of the edge-aware mean.
//
// P:243-245 define the mean with the indicator W_ij = delta{DT(z_i) - DT(z_j) <= r}; reading
// R25 takes it as the normalised box window on the guide's domain-transform axis,
//     zbar_i = (1/|N_i|) sum_{j in N_i} z_j,   N_i = { j : |T_j - T_i| <= r },
// N passes of rows then columns with r_i = radius_scale * sigma_i, and the support
// S = |N^x| |N^y| at r = radius_scale * sigma_s.
//
// Window membership is an integer decision: the increment d is evaluated in IEEE fp32 in
// the fixed order of R25 (no contraction, correctly rounded sqrt) and the DT axis is held
// in fixed point, q = rn(d * 2^16) (capped at 2^30), R = floor(r * 2^16); then the windows
// are exact integers.  They depend only on the guide, so dts_create computes them once:
//   K_B1 k_box_increments  q between each pixel and its left / upper neighbour
//   K_B2 k_box_windows     one outward walk per pixel and axis records the window edges of
//                          every radius (the radii are nested); packs lo | hi << 16 per pass
//                          and axis, and writes S = count_x * count_y
// Per pass (every iteration):
//   K_B3 k_box_row         a warp per row segment: the segment and its halo are staged in
//                          shared memory, an fp32 exclusive prefix inside 32-element blocks
//                          plus an fp64 prefix of the block totals give E(k) = sum_{j<k} x_j;
//                          zbar = (E(hi + 1) - E(lo)) / (hi - lo + 1)
//   K_B4 k_box_col         the same over a 32-column x (SEG + 2h)-row tile of a CTA (lane =
//                          column, coalesced 128-B rows)
// The halo makes the passes out of place (the solver ping-pongs two state buffers).
// Algorithmic bytes per pixel and pass: 4 C_t read + 4 window + 4 C_t write.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "dts_launch.h"

namespace dts {
namespace box {

constexpr uint32_t QMAX = 1u << 30;

// R25: d = sqrt(1 + k2 * sum_k (I_k(p) - I_k(p'))^2) in fp32, this order, no FMA
__device__ __forceinline__ uint32_t increment(const float* __restrict__ a, const float* __restrict__ b, int C,
                                              float k2) {
    float s = 0.0f;
    for (int k = 0; k < C; ++k) {
        const float diff = __fsub_rn(__ldg(a + k), __ldg(b + k));
        s = __fadd_rn(s, __fmul_rn(diff, diff));
    }
    const float v = __fadd_rn(1.0f, __fmul_rn(k2, s));
    const float d = __fsqrt_rn(v);
    const long long q = __float2ll_rn(__fmul_rn(d, 65536.0f));
    return q > (long long)QMAX ? QMAX : (uint32_t)q;
}

__global__ void __launch_bounds__(256) k_box_increments(const float* __restrict__ guide, int C, float k2, int64_t H,
                                                        int64_t W, int64_t pitch, uint32_t* __restrict__ qx,
                                                        uint32_t* __restrict__ qy) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (c >= W || r >= H) return;
    const float* p = guide + (r * W + c) * C;
    qx[r * pitch + c] = c == 0 ? 0u : increment(p, p - C, C, k2);
    qy[r * pitch + c] = r == 0 ? 0u : increment(p, p - W * C, C, k2);
}

// R25 quantisation of a channel sum s (the tail of increment() above)
__device__ __forceinline__ uint32_t quantise(float s, float k2) {
    const float v = __fadd_rn(1.0f, __fmul_rn(k2, s));
    const float d = __fsqrt_rn(v);
    const long long q = __float2ll_rn(__fmul_rn(d, 65536.0f));
    return q > (long long)QMAX ? QMAX : (uint32_t)q;
}

// K_B1 for C = 4Q channels (16-B aligned guide): the layout of the guide-derivative kernel
// (k_misc.cu k_guide_deriv_vec).  A thread walks 32 rows of one column; a pixel's channels
// arrive as Q float4 loads, the row above stays in registers, the next row is in flight;
// a warp covers 31 output columns and lane 0 loads the column before them, so every left
// neighbour comes by shuffle.  The channel sums keep increment()'s order and rounding.
constexpr int BI_ROWS = 32, BI_COLS = 8 * 31;
template <int Q>
__global__ void __launch_bounds__(256) k_box_increments_vec(const float* __restrict__ guide, float k2, int64_t H,
                                                            int64_t W, int64_t pitch, uint32_t* __restrict__ qx,
                                                            uint32_t* __restrict__ qy) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * BI_COLS + warp * 31 + lane - 1;  // lane 0: c0 - 1
    const int64_t rbeg = (int64_t)blockIdx.y * BI_ROWS;
    const int64_t rend = min(rbeg + (int64_t)BI_ROWS, H);
    const bool writer = lane > 0 && c < W;
    const int64_t cc = c < 0 ? 0 : (c >= W ? W - 1 : c);  // clamped: shuffles stay defined
    auto px = [&](int64_t r) { return reinterpret_cast<const float4*>(guide + (r * W + cc) * (4 * Q)); };
    float4 up[Q], cur[Q], ncur[Q];
    if (rbeg > 0) {
        const float4* pu = px(rbeg - 1);
#pragma unroll
        for (int q = 0; q < Q; ++q) up[q] = __ldg(pu + q);
    }
    {
        const float4* pc = px(rbeg);
#pragma unroll
        for (int q = 0; q < Q; ++q) cur[q] = __ldg(pc + q);
    }
    for (int64_t r = rbeg; r < rend; ++r) {
        if (r + 1 < rend) {
            const float4* pc = px(r + 1);
#pragma unroll
            for (int q = 0; q < Q; ++q) ncur[q] = __ldg(pc + q);
        }
        float sx = 0.0f, sy = 0.0f;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const float a[4] = {cur[q].x, cur[q].y, cur[q].z, cur[q].w};
            const float u[4] = {up[q].x, up[q].y, up[q].z, up[q].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // channel 4q + e, in order
                const float l = __shfl_up_sync(0xffffffffu, a[e], 1);
                const float dxv = __fsub_rn(a[e], l), dyv = __fsub_rn(a[e], u[e]);
                sx = __fadd_rn(sx, __fmul_rn(dxv, dxv));
                sy = __fadd_rn(sy, __fmul_rn(dyv, dyv));
            }
        }
        if (writer) {
            qx[r * pitch + c] = c == 0 ? 0u : quantise(sx, k2);
            qy[r * pitch + c] = r == 0 ? 0u : quantise(sy, k2);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            up[q] = cur[q];
            cur[q] = ncur[q];
        }
    }
}

constexpr int MAXR = 17;  // N <= 16 passes + the support radius
struct Radii {
    long long R[MAXR];  // R[0..N-1]: passes, R[N]: support
    int n;
    long long Rmax;
};

// walk from position i along a line (q at stride) in one direction; off[k] = number of
// steps whose cumulative distance stays <= R[k]
template <int DIR>
__device__ __forceinline__ void walk(const uint32_t* __restrict__ q, int64_t stride, int64_t i, int64_t n,
                                     const Radii& rd, int* off) {
#pragma unroll 1
    for (int k = 0; k < rd.n; ++k) off[k] = 0;
    long long dist = 0;
    int steps = 0;
    int64_t j = i;
#pragma unroll 1
    while (DIR < 0 ? j > 0 : j + 1 < n) {
        const long long nd = dist + (long long)__ldg(q + (DIR < 0 ? j : j + 1) * stride);
        if (nd > rd.Rmax) break;
        dist = nd;
        ++steps;
        j += DIR;
#pragma unroll 1
        for (int k = 0; k < rd.n; ++k)
            if (dist <= rd.R[k]) off[k] = steps;
    }
}

// the same walk with the radius count NR fixed at compile time: off[] stays in registers (the
// generic walk keeps it in local memory, which is what bounded K_B2: 2.45 ms on C4)
template <int NR, int DIR>
__device__ __forceinline__ void walk_t(const uint32_t* __restrict__ q, int64_t stride, int64_t i, int64_t n,
                                       const Radii& rd, int* off) {
#pragma unroll
    for (int k = 0; k < NR; ++k) off[k] = 0;
    long long dist = 0;
    int steps = 0;
    int64_t j = i;
#pragma unroll 1
    while (DIR < 0 ? j > 0 : j + 1 < n) {
        const long long nd = dist + (long long)__ldg(q + (DIR < 0 ? j : j + 1) * stride);
        if (nd > rd.Rmax) break;
        dist = nd;
        ++steps;
        j += DIR;
#pragma unroll
        for (int k = 0; k < NR; ++k)
            if (dist <= rd.R[k]) off[k] = steps;
    }
}

template <int NR>
__global__ void __launch_bounds__(256) k_box_windows_t(const uint32_t* __restrict__ qx, const uint32_t* __restrict__ qy,
                                                       int64_t H, int64_t W, int64_t pitch, int64_t plane, Radii rd,
                                                       uint32_t* __restrict__ win, float* __restrict__ S) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (c >= W || r >= H) return;
    int lo[NR], hi[NR];
    constexpr int np = NR - 1;
    walk_t<NR, -1>(qx + r * pitch, 1, c, W, rd, lo);
    walk_t<NR, +1>(qx + r * pitch, 1, c, W, rd, hi);
#pragma unroll
    for (int k = 0; k < np; ++k) win[(2 * k) * plane + r * pitch + c] = (uint32_t)lo[k] | ((uint32_t)hi[k] << 16);
    const float cx = (float)(lo[np] + hi[np] + 1);
    walk_t<NR, -1>(qy + c, pitch, r, H, rd, lo);
    walk_t<NR, +1>(qy + c, pitch, r, H, rd, hi);
#pragma unroll
    for (int k = 0; k < np; ++k) win[(2 * k + 1) * plane + r * pitch + c] = (uint32_t)lo[k] | ((uint32_t)hi[k] << 16);
    S[r * pitch + c] = cx * (float)(lo[np] + hi[np] + 1);
}

__global__ void __launch_bounds__(256) k_box_windows(const uint32_t* __restrict__ qx, const uint32_t* __restrict__ qy,
                                                     int64_t H, int64_t W, int64_t pitch, int64_t plane, Radii rd,
                                                     uint32_t* __restrict__ win, float* __restrict__ S) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (c >= W || r >= H) return;
    int lo[MAXR], hi[MAXR];
    const int np = rd.n - 1;
    // rows
    walk<-1>(qx + r * pitch, 1, c, W, rd, lo);
    walk<+1>(qx + r * pitch, 1, c, W, rd, hi);
#pragma unroll 1
    for (int k = 0; k < np; ++k) win[(2 * k) * plane + r * pitch + c] = (uint32_t)lo[k] | ((uint32_t)hi[k] << 16);
    const float cx = (float)(lo[np] + hi[np] + 1);
    // columns
    walk<-1>(qy + c, pitch, r, H, rd, lo);
    walk<+1>(qy + c, pitch, r, H, rd, hi);
#pragma unroll 1
    for (int k = 0; k < np; ++k) win[(2 * k + 1) * plane + r * pitch + c] = (uint32_t)lo[k] | ((uint32_t)hi[k] << 16);
    S[r * pitch + c] = cx * (float)(lo[np] + hi[np] + 1);
}

__device__ __forceinline__ float warp_incl_scan(float v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// window mean from the staged prefix E(k) = Pb[k >> 5] + pe[k] (pe: exclusive prefix inside
// the 32-block, so pe = 0 at a block start; Pb: fp64 exclusive prefix of the block totals):
// the whole-block part of the sum in fp64, rounded once, the in-block parts in fp32
template <int STRIDE>
__device__ __forceinline__ float window_mean(const float* pe, const double* pb, int li, int hi1, int cnt) {
    const float whole = (float)(pb[(hi1 >> 5) * STRIDE] - pb[(li >> 5) * STRIDE]);
    const float sum = whole + (pe[hi1 * STRIDE] - pe[li * STRIDE]);
    float rc;  // 1 / cnt, <= 1 ulp (cnt >= 1)
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"((float)cnt));
    return sum * rc;
}

// one output: decode the packed window of local index kl and form its mean
template <int STRIDE>
__device__ __forceinline__ float box_out(const float* pe, const double* pb, int kl, uint32_t w) {
    const int lo = (int)(w & 0xffffu), hi = (int)(w >> 16);
    return window_mean<STRIDE>(pe, pb, kl - lo, kl + hi + 1, lo + hi + 1);
}

// shared memory of one warp of k_box_row: pe[lpad] floats + pb[lpad / 32] doubles, 16-B multiple
__host__ __device__ constexpr size_t row_warp_bytes(int lpad) {
    return ((size_t)lpad * 4 + (size_t)(lpad / 32) * 8 + 15) & ~(size_t)15;
}

struct RowArgs {
    const float* in;
    float* out;
    const uint32_t* win;
    int64_t H, W, pitch, plane;
    int Ct, h, seg, nseg, lpad;  // lpad: staged floats per warp (multiple of 128, >= 32 (nblk + 1))
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

constexpr int WB = 8;  // window loads in flight per lane

// K_B3: a warp per (row, segment); channels loop inside.  Shared memory per warp: pe[lpad]
// floats and pb[lpad / 32] doubles.  Staged values at or beyond b (pad columns, stale
// shared memory) are never inside a window and enter only prefixes no window reads.
__global__ void __launch_bounds__(256) k_box_row(RowArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const size_t per_warp = row_warp_bytes(p.lpad);
    float* pe = reinterpret_cast<float*>(smem_raw + per_warp * wid);
    double* pb = reinterpret_cast<double*>(smem_raw + per_warp * wid + (size_t)p.lpad * 4);
    const int64_t ntask = p.H * p.nseg;
    const int sub = lane & 7;
    for (int64_t task = (int64_t)blockIdx.x * nw + wid; task < ntask; task += (int64_t)gridDim.x * nw) {
        const int64_t r = task / p.nseg;
        const int64_t c0 = (task - r * p.nseg) * p.seg;
        const int64_t c1 = c0 + p.seg < p.W ? c0 + p.seg : p.W;
        const int64_t a = c0 - p.h > 0 ? c0 - p.h : 0;
        const int64_t b = c1 + p.h < p.W ? c1 + p.h : p.W;
        const int64_t a4 = a & ~(int64_t)3;  // 16-B aligned start (rows are 128-B aligned)
        const int L = (int)(b - a4);
        const int L4 = (L + 3) & ~3;         // staged floats (a4 + L4 <= pitch)
        const int nchunk = ((L >> 5) + 1 + 3) >> 2;  // 128-float chunks covering blocks 0..nblk
        const int n = (int)(c1 - c0), k0l = (int)(c0 - a4);  // outputs, local index of the first
        const uint32_t* wrow = p.win + r * p.pitch + c0;
        for (int ch = 0; ch < p.Ct; ++ch) {
            const float* xr = p.in + ch * p.plane + r * p.pitch + a4;
            for (int e = lane * 4; e < L4; e += 128) cp_async16(pe + e, xr + e);
            uint32_t w[WB];  // first window batch in flight during the scan
#pragma unroll
            for (int u = 0; u < WB; ++u) w[u] = (lane + 32 * u < n) ? __ldg(wrow + lane + 32 * u) : 0u;
            cp_async_wait_all();
            __syncwarp();
            // exclusive prefix inside 32-blocks: lane holds 4 consecutive floats, 8 lanes a
            // block (segmented shuffle scan); block totals -> fp64 exclusive prefix
            double run = 0.0;
            for (int c = 0; c < nchunk; ++c) {
                float4 v = *reinterpret_cast<const float4*>(pe + c * 128 + lane * 4);
                const float s1 = v.x + v.y, s2 = s1 + v.z, t = s2 + v.w;
                float inc = t;
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    const float nb = __shfl_up_sync(0xffffffffu, inc, o);
                    if (sub >= o) inc += nb;
                }
                float ex = __shfl_up_sync(0xffffffffu, inc, 1);
                if (sub == 0) ex = 0.f;
                *reinterpret_cast<float4*>(pe + c * 128 + lane * 4) = make_float4(ex, ex + v.x, ex + s1, ex + s2);
                const float t0 = __shfl_sync(0xffffffffu, inc, 7), t1 = __shfl_sync(0xffffffffu, inc, 15);
                const float t2 = __shfl_sync(0xffffffffu, inc, 23), t3 = __shfl_sync(0xffffffffu, inc, 31);
                const double p1 = run + (double)t0, p2 = p1 + (double)t1, p3 = p2 + (double)t2;
                if (lane < 4) pb[c * 4 + lane] = lane == 0 ? run : lane == 1 ? p1 : lane == 2 ? p2 : p3;
                run = p3 + (double)t3;
            }
            __syncwarp();
            float* orow = p.out + ch * p.plane + r * p.pitch + c0 + lane;
            const uint32_t* wl = wrow + lane;
            for (int j0 = 0; j0 < n; j0 += 32 * WB) {  // j0: warp-uniform batch start
                uint32_t wn[WB];  // next batch
                const int jn = j0 + 32 * WB;
                if (jn + 32 * WB <= n) {
#pragma unroll
                    for (int u = 0; u < WB; ++u) wn[u] = __ldg(wl + jn + 32 * u);
                } else {
#pragma unroll
                    for (int u = 0; u < WB; ++u) wn[u] = (jn + 32 * u + lane < n) ? __ldg(wl + jn + 32 * u) : 0u;
                }
                const int kb = k0l + j0 + lane;
                if (j0 + 32 * WB <= n) {
#pragma unroll
                    for (int u = 0; u < WB; ++u) orow[j0 + 32 * u] = box_out<1>(pe, pb, kb + 32 * u, w[u]);
                } else {
#pragma unroll
                    for (int u = 0; u < WB; ++u)
                        if (j0 + 32 * u + lane < n) orow[j0 + 32 * u] = box_out<1>(pe, pb, kb + 32 * u, w[u]);
                }
#pragma unroll
                for (int u = 0; u < WB; ++u) w[u] = wn[u];
            }
            __syncwarp();
        }
    }
}

struct ColArgs {
    const float* in;
    float* out;
    const uint32_t* win;
    int64_t H, W, pitch, plane;
    int Ct, h, seg, nseg, ntc, lpad;  // lpad: staged rows (multiple of 32) + 32
};

// K_B4: a CTA per (32-column tile, row segment); lane = column.  Shared memory:
// xs[lpad][32] floats (row-major, one 128-B row per image row) + pb[lpad/32][32] doubles.
__global__ void __launch_bounds__(256) k_box_col(ColArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* xs = reinterpret_cast<float*>(smem_raw);
    double* pb = reinterpret_cast<double*>(smem_raw + (size_t)p.lpad * 128);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t ntask = (int64_t)p.ntc * p.nseg;
    const int64_t pitch = p.pitch;
    const int64_t wstep = (int64_t)nw * pitch;  // rows nw apart
    for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
        const int64_t tc = task % p.ntc;  // consecutive CTAs take neighbouring column tiles
        const int64_t r0 = (task / p.ntc) * p.seg;
        const int64_t r1 = r0 + p.seg < p.H ? r0 + p.seg : p.H;
        const int64_t c0 = tc * 32;
        const int64_t a = r0 - p.h > 0 ? r0 - p.h : 0;
        const int64_t b = r1 + p.h < p.H ? r1 + p.h : p.H;
        const int L = (int)(b - a);
        const int nblk = (L + 31) >> 5;
        const int n = (int)(r1 - r0), k0l = (int)(r0 - a);
        const bool col_ok = c0 + lane < p.W;
        const uint32_t* wt = p.win + r0 * pitch + c0 + lane;
        for (int ch = 0; ch < p.Ct; ++ch) {
            const float* xt = p.in + ch * p.plane + a * p.pitch + c0;
            // stage rows [a, b) (8 x 16 B per row); rows L..32 nblk - 1 are never read by a
            // window; row 32 nblk (block start: exclusive prefix 0) closes the last block
            for (int e = threadIdx.x; e < L * 8; e += blockDim.x) {
                const int row = e >> 3, q4 = (e & 7) * 4;
                cp_async16(xs + row * 32 + q4, xt + (int64_t)row * p.pitch + q4);
            }
            if (threadIdx.x < 32) xs[nblk * 32 * 32 + threadIdx.x] = 0.f;  // pe at row 32 nblk
            uint32_t w[WB];  // first window batch in flight during the scan
            const uint32_t* wq = wt + (int64_t)wid * pitch;
#pragma unroll
            for (int u = 0; u < WB; ++u) w[u] = (col_ok && wid + nw * u < n) ? __ldg(wq + u * wstep) : 0u;
            cp_async_wait_all();
            __syncthreads();
            // exclusive prefix of each 32-row block of every column (fp32), block totals
            for (int j = wid; j < nblk; j += nw) {
                float run = 0.f;
                float* col = xs + j * 32 * 32 + lane;
                float v[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = col[k * 32];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    col[k * 32] = run;
                    run += v[k];
                }
                pb[j * 32 + lane] = (double)run;
            }
            __syncthreads();
            if (wid == 0) {  // exclusive prefix of the block totals (fp64)
                double run = 0.0;
                for (int j = 0; j < nblk; ++j) {
                    const double t = pb[j * 32 + lane];
                    pb[j * 32 + lane] = run;
                    run += t;
                }
                pb[nblk * 32 + lane] = run;
            }
            __syncthreads();
            if (col_ok) {
                float* oq = p.out + ch * p.plane + (r0 + wid) * pitch + c0 + lane;
                for (int j0 = 0; j0 < n; j0 += nw * WB) {  // warp rows j0 + wid + nw u
                    uint32_t wn[WB];
                    wq += (int64_t)WB * wstep;
                    const int jn = j0 + nw * WB + wid;
                    if (jn + nw * (WB - 1) < n) {
#pragma unroll
                        for (int u = 0; u < WB; ++u) wn[u] = __ldg(wq + u * wstep);
                    } else {
#pragma unroll
                        for (int u = 0; u < WB; ++u) wn[u] = (jn + nw * u < n) ? __ldg(wq + u * wstep) : 0u;
                    }
                    const int kb = k0l + j0 + wid;
                    if (j0 + wid + nw * (WB - 1) < n) {
#pragma unroll
                        for (int u = 0; u < WB; ++u) oq[u * wstep] = box_out<32>(xs + lane, pb + lane, kb + nw * u, w[u]);
                    } else {
#pragma unroll
                        for (int u = 0; u < WB; ++u)
                            if (j0 + wid + nw * u < n) oq[u * wstep] = box_out<32>(xs + lane, pb + lane, kb + nw * u, w[u]);
                    }
                    oq += (int64_t)WB * wstep;
#pragma unroll
                    for (int u = 0; u < WB; ++u) w[u] = wn[u];
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------------------
// host side

static int occupancy(const void* fn, int threads, size_t smem) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace box

cudaError_t launch_box_increments(const float* guide, int C, float k2, const Geometry& g, uint32_t* qx, uint32_t* qy,
                                  cudaStream_t s) {
    dim3 grid((unsigned)((g.W + 255) / 256), (unsigned)g.H);
    if ((C == 4 || C == 8 || C == 16) && (uintptr_t)guide % 16 == 0) {
        const dim3 gv((unsigned)((g.W + 1 + box::BI_COLS - 1) / box::BI_COLS),
                      (unsigned)((g.H + box::BI_ROWS - 1) / box::BI_ROWS));
        if (C == 4) box::k_box_increments_vec<1><<<gv, 256, 0, s>>>(guide, k2, g.H, g.W, g.pitch, qx, qy);
        if (C == 8) box::k_box_increments_vec<2><<<gv, 256, 0, s>>>(guide, k2, g.H, g.W, g.pitch, qx, qy);
        if (C == 16) box::k_box_increments_vec<4><<<gv, 256, 0, s>>>(guide, k2, g.H, g.W, g.pitch, qx, qy);
        return cudaGetLastError();
    }
    box::k_box_increments<<<grid, 256, 0, s>>>(guide, C, k2, g.H, g.W, g.pitch, qx, qy);
    return cudaGetLastError();
}

cudaError_t launch_box_windows(const uint32_t* qx, const uint32_t* qy, const Geometry& g, const long long* R, int nR,
                               uint32_t* win, float* S, cudaStream_t s) {
    if (nR < 2 || nR > box::MAXR) return cudaErrorInvalidValue;
    box::Radii rd = {};
    rd.n = nR;
    rd.Rmax = 0;
    for (int k = 0; k < nR; ++k) {
        rd.R[k] = R[k];
        if (R[k] > rd.Rmax) rd.Rmax = R[k];
    }
    dim3 grid((unsigned)((g.W + 255) / 256), (unsigned)g.H);
    switch (nR) {  // N = 1..4 passes (+ the support radius): registers; otherwise the generic walk
        case 2: box::k_box_windows_t<2><<<grid, 256, 0, s>>>(qx, qy, g.H, g.W, g.pitch, g.plane, rd, win, S); break;
        case 3: box::k_box_windows_t<3><<<grid, 256, 0, s>>>(qx, qy, g.H, g.W, g.pitch, g.plane, rd, win, S); break;
        case 4: box::k_box_windows_t<4><<<grid, 256, 0, s>>>(qx, qy, g.H, g.W, g.pitch, g.plane, rd, win, S); break;
        case 5: box::k_box_windows_t<5><<<grid, 256, 0, s>>>(qx, qy, g.H, g.W, g.pitch, g.plane, rd, win, S); break;
        default: box::k_box_windows<<<grid, 256, 0, s>>>(qx, qy, g.H, g.W, g.pitch, g.plane, rd, win, S);
    }
    return cudaGetLastError();
}

cudaError_t plan_box(const Geometry& g, long long R, int num_sms, BoxPlan* plan) {
    const long long hmax = R >> 16;  // every step is >= 2^16 (d >= 1): no window is wider
    plan->hx = (int)(hmax < g.W - 1 ? hmax : g.W - 1);
    plan->hy = (int)(hmax < g.H - 1 ? hmax : g.H - 1);
    // rows: a warp per segment of <= 1024 outputs plus the halo
    // segments of 1024 outputs (measured on C4: 1024 -> 0.221 ms, 2048 -> 0.246, 512 -> 0.253)
    plan->row_seg = (int)(g.W < 1024 ? g.W : 1024);
    plan->row_nseg = (int)((g.W + plan->row_seg - 1) / plan->row_seg);
    long long lrow = (long long)plan->row_seg + 2LL * plan->hx + 3;
    if (lrow > g.W + 3) lrow = g.W + 3;
    plan->row_lpad = (int)((((lrow >> 5) + 4) >> 2) * 128);  // 128-float chunks covering blocks 0..L/32
    const size_t pw = box::row_warp_bytes(plan->row_lpad);
    if (pw > 200 * 1024) return cudaErrorInvalidValue;
    int warps = (int)((110 * 1024) / pw);
    warps = warps < 1 ? 1 : warps > 8 ? 8 : warps;
    plan->row_threads = warps * 32;
    plan->row_smem = pw * warps;
    // the attribute is per function, shared by the plans of all passes: set it to the
    // opt-in maximum once, so that no plan lowers another's limit
    int optin = 0, dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    if (plan->row_smem > (size_t)optin) return cudaErrorInvalidValue;
    const void* frow = reinterpret_cast<const void*>(box::k_box_row);
    if ((e = cudaFuncSetAttribute(frow, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess) return e;
    const int orow = box::occupancy(frow, plan->row_threads, plan->row_smem);
    if (orow < 1) return cudaErrorInvalidValue;
    const long long rtasks = (g.H * plan->row_nseg + warps - 1) / warps;
    plan->row_grid = (int)(rtasks < (long long)num_sms * orow ? rtasks : (long long)num_sms * orow);
    // columns: a CTA per 32-column tile x segment
    // ~480 staged rows per tile (measured on C4: 480 -> 0.258 ms, 736 -> 0.269, 352 -> 0.276)
    long long seg = (480 - 2LL * plan->hy) / 32 * 32;
    if (seg < 32) seg = 32;
    if (seg > g.H) seg = g.H;
    plan->col_seg = (int)seg;
    plan->col_nseg = (int)((g.H + seg - 1) / seg);
    plan->col_ntc = (int)((g.W + 31) / 32);
    long long lcol = seg + 2LL * plan->hy;
    if (lcol > g.H) lcol = g.H;
    plan->col_lpad = (int)((lcol + 31) / 32 * 32 + 32);
    plan->col_smem = (size_t)plan->col_lpad * 128 + (size_t)plan->col_lpad / 32 * 32 * 8;
    if (plan->col_smem > (size_t)optin) return cudaErrorInvalidValue;
    const void* fcol = reinterpret_cast<const void*>(box::k_box_col);
    if ((e = cudaFuncSetAttribute(fcol, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess) return e;
    const int ocol = box::occupancy(fcol, 256, plan->col_smem);
    if (ocol < 1) return cudaErrorInvalidValue;
    const long long ctasks = (long long)plan->col_ntc * plan->col_nseg;
    plan->col_grid = (int)(ctasks < (long long)num_sms * ocol ? ctasks : (long long)num_sms * ocol);
    return cudaSuccess;
}

cudaError_t launch_box_row(const BoxPlan& plan, const Geometry& g, int Ct, const float* in, float* out,
                           const uint32_t* win, cudaStream_t s) {
    box::RowArgs a;
    a.in = in;
    a.out = out;
    a.win = win;
    a.H = g.H;
    a.W = g.W;
    a.pitch = g.pitch;
    a.plane = g.plane;
    a.Ct = Ct;
    a.h = plan.hx;
    a.seg = plan.row_seg;
    a.nseg = plan.row_nseg;
    a.lpad = plan.row_lpad;
    box::k_box_row<<<plan.row_grid, plan.row_threads, plan.row_smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_box_col(const BoxPlan& plan, const Geometry& g, int Ct, const float* in, float* out,
                           const uint32_t* win, cudaStream_t s) {
    box::ColArgs a;
    a.in = in;
    a.out = out;
    a.win = win;
    a.H = g.H;
    a.W = g.W;
    a.pitch = g.pitch;
    a.plane = g.plane;
    a.Ct = Ct;
    a.h = plan.hy;
    a.seg = plan.col_seg;
    a.nseg = plan.col_nseg;
    a.ntc = plan.col_ntc;
    a.lpad = plan.col_lpad;
    box::k_box_col<<<plan.col_grid, 256, plan.col_smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace dts
