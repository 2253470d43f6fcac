// k_misc.cu -- K1 (guide derivative) and K6 (solve prologue) for sm_100a.
#include "dts_device.cuh"
#include "dts_launch.h"

#include <mutex>
#include <utility>
#include <vector>

namespace dts {

// K1: domain-transform increments between adjacent pixels (Eqs. 8-9 with
// the square restored, R1; sigma scaling R2):
//     d_x[r][c] = sqrt(1 + (sigma_s/sigma_r)^2 sum_k (I[r][c][k] - I[r][c-1][k])^2), d_x[r][0] = +inf
//     d_y[r][c] likewise with row r-1, d_y[0][c] = +inf; columns c >= W (pitch padding) = +inf.
// A CTA owns a strip of 256 pixels (+1 on the left) and walks KROWS rows down it.
// Each HWC row strip is one contiguous span of 257*C floats: it is loaded with
// fully coalesced, independent loads (all in flight at once), parked in shared
// memory with a conflict-free odd pixel stride, and the previous row stays
// resident, so the guide is read from HBM once (plus 1/KROWS re-read of a row).
constexpr int DERIV_STRIP = 256;
constexpr int DERIV_ROWS = 32;

template <int CT>  // CT = channel count (0: runtime C)
__global__ void __launch_bounds__(DERIV_STRIP) k_guide_deriv(const float* __restrict__ guide, int Crt, float ratio2,
                                                             Geometry g, float* __restrict__ dx,
                                                             float* __restrict__ dy, float* __restrict__ a1y,
                                                             float kc0) {
    const int C = CT > 0 ? CT : Crt;
    const int CS = C | 1;  // odd pixel stride in shared memory -> conflict-free reads
    extern __shared__ float sm[];
    float* buf[2] = {sm, sm + (DERIV_STRIP + 1) * CS};
    const int64_t c0 = (int64_t)blockIdx.x * DERIV_STRIP;  // first pixel of the strip
    const int64_t rbeg = (int64_t)blockIdx.y * DERIV_ROWS;
    const int64_t rend = min(rbeg + DERIV_ROWS, g.H);
    const int t = threadIdx.x;
    const int64_t cfirst = c0 > 0 ? c0 - 1 : 0;               // first pixel loaded
    const int64_t clast = min(c0 + DERIV_STRIP, g.W);          // one past the last
    const int64_t npx = clast > cfirst ? clast - cfirst : 0;
    const int off = c0 > 0 ? 0 : 1;                            // smem pixel slot of `cfirst`
    const int64_t n = npx * C;

    // register-staged, software-pipelined row loads: row r+1 is in flight while row r computes
    constexpr int NPER = CT > 0 ? (CT * (DERIV_STRIP + 1) + DERIV_STRIP - 1) / DERIV_STRIP : 1;
    float v[NPER];
    auto fetch = [&](int64_t r) {
        const float* src = guide + (r * g.W + cfirst) * C;
#pragma unroll
        for (int u = 0; u < NPER; ++u) {
            const int64_t e = t + (int64_t)u * DERIV_STRIP;
            v[u] = e < n ? __ldg(src + e) : 0.f;
        }
    };
    auto park = [&](float* dst) {
#pragma unroll
        for (int u = 0; u < NPER; ++u) {
            const int64_t e = t + (int64_t)u * DERIV_STRIP;
            if (e < n) {
                const int px = (int)(e / C), k = (int)(e - (int64_t)px * C);
                dst[(px + off) * CS + k] = v[u];
            }
        }
    };
    auto load_row_slow = [&](int64_t r, float* dst) {  // runtime C
        const float* src = guide + (r * g.W + cfirst) * C;
        for (int64_t e = t; e < n; e += DERIV_STRIP) {
            const int px = (int)(e / C), k = (int)(e - (int64_t)px * C);
            dst[(px + off) * CS + k] = __ldg(src + e);
        }
    };

    const int64_t c = c0 + t;  // this thread's pixel; smem slot t + 1
    int cur = 0;
    if (rbeg > 0) {
        if constexpr (CT > 0) {
            fetch(rbeg - 1);
            park(buf[1]);
        } else {
            load_row_slow(rbeg - 1, buf[1]);
        }
    }
    if constexpr (CT > 0) fetch(rbeg);
    for (int64_t r = rbeg; r < rend; ++r) {
        if constexpr (CT > 0) {
            park(buf[cur]);
        } else {
            load_row_slow(r, buf[cur]);
        }
        __syncthreads();
        if constexpr (CT > 0) {
            if (r + 1 < rend) fetch(r + 1);
        }
        if (c < g.pitch) {
            float ox = __int_as_float(0x7f800000), oy = __int_as_float(0x7f800000);
            if (c < g.W) {
                const float* pc = buf[cur] + (t + 1) * CS;
                const float* pl = buf[cur] + t * CS;
                const float* pu = buf[cur ^ 1] + (t + 1) * CS;
                float sx = 0.f, sy = 0.f;
                for (int k = 0; k < C; ++k) {
                    const float x = pc[k];
                    const float ex = x - pl[k], ey = x - pu[k];
                    sx = fmaf(ex, ex, sx);
                    sy = fmaf(ey, ey, sy);
                }
                if (c > 0) ox = sqrtf(fmaf(ratio2, sx, 1.f));
                if (r > 0) oy = sqrtf(fmaf(ratio2, sy, 1.f));
            }
            dx[r * g.pitch + c] = ox;
            dy[r * g.pitch + c] = oy;
            if (a1y) a1y[r * g.pitch + c] = coef_from_d(oy, kc0);  // pass-1 column coefficient
        }
        cur ^= 1;
        __syncthreads();
    }
}

// K1 for C % 4 == 0 (e.g. the 16-band satellite guide): one thread per pixel column,
// walking DERIV_ROWS rows; each pixel's C channels arrive as C/4 float4 loads (a warp
// covers one contiguous 32*C-float span), the previous row stays in registers, and the
// next row's loads are issued before the current row's arithmetic.  Each warp covers 31
// output columns: lane 0 loads the column before them (the left neighbour of lane 1,
// handed over by a shuffle like every lane's) and writes nothing, so every lane keeps only
// up / cur / next-row registers.
constexpr int DERIV_VEC_COLS = 8 * 31;  // output columns per 256-thread block
template <int Q>  // Q = C / 4
__global__ void __launch_bounds__(256) k_guide_deriv_vec(const float* __restrict__ guide, float ratio2, Geometry g,
                                                         float* __restrict__ dx, float* __restrict__ dy,
                                                         float* __restrict__ a1y, float kc0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * DERIV_VEC_COLS + warp * 31 + lane - 1;  // lane 0: c0 - 1
    const int64_t rbeg = (int64_t)blockIdx.y * DERIV_ROWS;
    const int64_t rend = min(rbeg + (int64_t)DERIV_ROWS, g.H);
    const bool writer = lane > 0 && c < g.pitch;
    const float inf = __int_as_float(0x7f800000);
    if (c >= g.W || c < 0) {  // padding columns (writers) or the column before the image (lane 0)
        if (writer)
            for (int64_t r = rbeg; r < rend; ++r) {
                dx[r * g.pitch + c] = inf;
                dy[r * g.pitch + c] = inf;
                if (a1y) a1y[r * g.pitch + c] = 0.f;
            }
        // keep the warp's shuffles well-defined: fall through with a clamped column
    }
    const int64_t cc = c < 0 ? 0 : (c >= g.W ? g.W - 1 : c);
    auto px = [&](int64_t r) { return reinterpret_cast<const float4*>(guide + (r * g.W + cc) * (4 * Q)); };
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
        if (r + 1 < rend) {  // next row in flight during this row's arithmetic
            const float4* pc = px(r + 1);
#pragma unroll
            for (int q = 0; q < Q; ++q) ncur[q] = __ldg(pc + q);
        }
        float sx = 0.f, sy = 0.f;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const float lx = __shfl_up_sync(0xffffffffu, cur[q].x, 1), ly = __shfl_up_sync(0xffffffffu, cur[q].y, 1);
            const float lz = __shfl_up_sync(0xffffffffu, cur[q].z, 1), lw = __shfl_up_sync(0xffffffffu, cur[q].w, 1);
            const float ax = cur[q].x - lx, ay = cur[q].y - ly, az = cur[q].z - lz, aw = cur[q].w - lw;
            const float bx = cur[q].x - up[q].x, by = cur[q].y - up[q].y, bz = cur[q].z - up[q].z,
                        bw = cur[q].w - up[q].w;
            sx = fmaf(ax, ax, fmaf(ay, ay, fmaf(az, az, fmaf(aw, aw, sx))));
            sy = fmaf(bx, bx, fmaf(by, by, fmaf(bz, bz, fmaf(bw, bw, sy))));
        }
        if (writer && c < g.W) {
            dx[r * g.pitch + c] = c > 0 ? sqrtf(fmaf(ratio2, sx, 1.f)) : inf;
            const float oy = r > 0 ? sqrtf(fmaf(ratio2, sy, 1.f)) : inf;
            dy[r * g.pitch + c] = oy;
            if (a1y) a1y[r * g.pitch + c] = coef_from_d(oy, kc0);  // pass-1 column coefficient
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            up[q] = cur[q];
            cur[q] = ncur[q];
        }
    }
}

cudaError_t launch_guide_deriv(const float* guide, int C, float ratio2, const Geometry& g, float* dx, float* dy,
                               cudaStream_t s, float* a1y, float kc0) {
    if ((C == 4 || C == 8 || C == 16) && ((uintptr_t)guide % 16 == 0)) {
        dim3 block(256);
        dim3 grid((unsigned)((g.pitch + DERIV_VEC_COLS - 1) / DERIV_VEC_COLS),
                  (unsigned)((g.H + DERIV_ROWS - 1) / DERIV_ROWS));
        if (C == 4) k_guide_deriv_vec<1><<<grid, block, 0, s>>>(guide, ratio2, g, dx, dy, a1y, kc0);
        if (C == 8) k_guide_deriv_vec<2><<<grid, block, 0, s>>>(guide, ratio2, g, dx, dy, a1y, kc0);
        if (C == 16) k_guide_deriv_vec<4><<<grid, block, 0, s>>>(guide, ratio2, g, dx, dy, a1y, kc0);
        return cudaGetLastError();
    }
    dim3 block(DERIV_STRIP);
    dim3 grid((unsigned)((g.pitch + DERIV_STRIP - 1) / DERIV_STRIP), (unsigned)((g.H + DERIV_ROWS - 1) / DERIV_ROWS));
    const size_t smem = 2 * (size_t)(DERIV_STRIP + 1) * (C | 1) * sizeof(float);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    switch (C) {
#define DTS_DERIV_CASE(K)                                                                              \
    case K: {                                                                                         \
        cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k_guide_deriv<K>), smem);      \
        if (e != cudaSuccess) return e;                                                               \
        k_guide_deriv<K><<<grid, block, smem, s>>>(guide, C, ratio2, g, dx, dy, a1y, kc0);            \
        break;                                                                                        \
    }
        DTS_DERIV_CASE(1)
        DTS_DERIV_CASE(3)
        DTS_DERIV_CASE(4)
        DTS_DERIV_CASE(16)
        default: {
            cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k_guide_deriv<0>), smem);
            if (e != cudaSuccess) return e;
            k_guide_deriv<0><<<grid, block, smem, s>>>(guide, C, ratio2, g, dx, dy, a1y, kc0);
        }
#undef DTS_DERIV_CASE
    }
    return cudaGetLastError();
}

// K6: planar state from the HWC target, chat = c / S (R7).  One thread per 4
// consecutive pixels of a row: float4 stores of Z, T, chat (and float4 loads of the target
// and confidence when a row of them is 16-B aligned, i.e. W % 4 == 0 and C_t == 1).
template <bool VEC>
__global__ void __launch_bounds__(256) k_prologue(const float* __restrict__ target, const float* __restrict__ conf,
                                                  int Ct, Geometry g, const float* __restrict__ S,
                                                  const float* __restrict__ Sy, int support_mode,
                                                  float* __restrict__ Z, float* __restrict__ T,
                                                  float* __restrict__ chat) {
    pdl_wait();
    const int64_t per_row = g.pitch / 4;
    const int64_t n = g.H * per_row;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_row;
        const int64_t c4 = (i - r * per_row) * 4;
        if (c4 >= g.W) continue;
        const int64_t o = r * g.pitch + c4;
        const int64_t p = r * g.W + c4;
        float cv[4];
        if constexpr (VEC) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(conf + p));
            cv[0] = q.x; cv[1] = q.y; cv[2] = q.z; cv[3] = q.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) cv[u] = (c4 + u < g.W) ? __ldg(conf + p + u) : 0.f;
        }
        float4 sv = __ldg(reinterpret_cast<const float4*>(S + o));
        if (Sy) {  // support kept as its two separable factors: S = s_x s_y (R7)
            const float4 sy = __ldg(reinterpret_cast<const float4*>(Sy + o));
            sv = make_float4(sv.x * sy.x, sv.y * sy.y, sv.z * sy.z, sv.w * sy.w);
        }
        const float ss[4] = {sv.x, sv.y, sv.z, sv.w};
        float ch[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ch[u] = (c4 + u < g.W) ? (support_mode == 1 ? cv[u] : cv[u] / ss[u]) : 0.f;
        *reinterpret_cast<float4*>(chat + o) = make_float4(ch[0], ch[1], ch[2], ch[3]);
        for (int v = 0; v < Ct; ++v) {
            float tv[4];
            if constexpr (VEC) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(target + p));
                tv[0] = q.x; tv[1] = q.y; tv[2] = q.z; tv[3] = q.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) tv[u] = (c4 + u < g.W) ? __ldg(target + (p + u) * Ct + v) : 0.f;
            }
            const float4 t4 = make_float4(tv[0], tv[1], tv[2], tv[3]);
            *reinterpret_cast<float4*>(Z + v * g.plane + o) = t4;
            *reinterpret_cast<float4*>(T + v * g.plane + o) = t4;
        }
    }
}

cudaError_t launch_prologue(const float* target, const float* conf, int Ct, const Geometry& g, const float* S,
                            const float* Sy,
                            int support_mode, float* Z, float* T, float* chat, cudaStream_t s) {
    const int64_t n = g.H * (g.pitch / 4);
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    const bool vec = Ct == 1 && g.W % 4 == 0 && ((uintptr_t)target % 16 == 0) && ((uintptr_t)conf % 16 == 0);
    if (vec)
        return launch_pdl(k_prologue<true>, dim3((unsigned)blocks), dim3(256), 0, s, target, conf, Ct, g, S, Sy,
                          support_mode, Z, T, chat);
    return launch_pdl(k_prologue<false>, dim3((unsigned)blocks), dim3(256), 0, s, target, conf, Ct, g, S, Sy,
                      support_mode, Z, T, chat);
}

// K4b: the Eq. (3) step as a streaming kernel, used after the
// cluster column kernel:  Z <- Z - step [lambda (Z - zbar) + chat (Z - T)], zbar = X;
// on the last iteration the result goes to the HWC output instead of Z.
// One thread per 4 consecutive pixels of a row (float4 loads of every plane); the HWC output of
// those 4 pixels is 4 CT consecutive floats, written as CT float4 stores when 16-byte aligned.
template <int CT>
__global__ void __launch_bounds__(256) k_update(const float* __restrict__ X, float* __restrict__ Z,
                                                const float* __restrict__ T, const float* __restrict__ chat,
                                                Geometry g, float lam, float step, float* __restrict__ out_hwc,
                                                unsigned* __restrict__ resid) {
    pdl_wait();
    const int64_t per_row = g.pitch / 4;
    const int64_t n = g.H * per_row;
    float gmax = 0.f;  // ||g||_inf of this step (K8), when resid is requested
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_row;
        const int64_t c4 = (i - r * per_row) * 4;
        if (c4 >= g.W) continue;
        const int64_t o = r * g.pitch + c4;
        const float4 ch4 = __ldg(reinterpret_cast<const float4*>(chat + o));
        const float ch[4] = {ch4.x, ch4.y, ch4.z, ch4.w};
        float zn[4][CT];  // [pixel][channel]
#pragma unroll
        for (int v = 0; v < CT; ++v) {
            const int64_t ov = v * g.plane + o;
            const float4 zb4 = __ldg(reinterpret_cast<const float4*>(X + ov));
            const float4 zo4 = *reinterpret_cast<const float4*>(Z + ov);
            const float4 tv4 = __ldg(reinterpret_cast<const float4*>(T + ov));
            const float zb[4] = {zb4.x, zb4.y, zb4.z, zb4.w};
            const float zo[4] = {zo4.x, zo4.y, zo4.z, zo4.w};
            const float tv[4] = {tv4.x, tv4.y, tv4.z, tv4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float gr = fmaf(lam, zo[u] - zb[u], ch[u] * (zo[u] - tv[u]));  // Eq. (3)
                zn[u][v] = fmaf(-step, gr, zo[u]);
                if (resid && c4 + u < g.W) gmax = fmaxf(gmax, fabsf(gr));
            }
            if (!out_hwc) *reinterpret_cast<float4*>(Z + ov) = make_float4(zn[0][v], zn[1][v], zn[2][v], zn[3][v]);
        }
        if (out_hwc) {
            float* dst = out_hwc + (r * g.W + c4) * CT;
            if (c4 + 3 < g.W && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                const float* f = &zn[0][0];  // 4 CT consecutive values, pixel-major = HWC
#pragma unroll
                for (int q = 0; q < CT; ++q)
                    reinterpret_cast<float4*>(dst)[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (c4 + u < g.W) {
#pragma unroll
                        for (int v = 0; v < CT; ++v) dst[u * CT + v] = zn[u][v];
                    }
            }
        }
    }
    if (resid) {  // max is order-independent: the result is deterministic
        const unsigned m = __reduce_max_sync(FULL, __float_as_uint(gmax));
        if ((threadIdx.x & 31) == 0 && m) atomicMax(resid, m);
    }
}

cudaError_t launch_update(const float* X, float* Z, const float* T, const float* chat, int Ct, const Geometry& g,
                          float lam, float step, float* out_hwc, int num_sms, cudaStream_t s, unsigned* resid) {
    const int64_t n = g.H * (g.pitch / 4);
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const dim3 grid((unsigned)blocks), block(256);
    switch (Ct) {
        case 1: return launch_pdl(k_update<1>, grid, block, 0, s, X, Z, T, chat, g, lam, step, out_hwc, resid);
        case 2: return launch_pdl(k_update<2>, grid, block, 0, s, X, Z, T, chat, g, lam, step, out_hwc, resid);
        case 3: return launch_pdl(k_update<3>, grid, block, 0, s, X, Z, T, chat, g, lam, step, out_hwc, resid);
        case 4: return launch_pdl(k_update<4>, grid, block, 0, s, X, Z, T, chat, g, lam, step, out_hwc, resid);
    }
    return cudaErrorInvalidValue;
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

__global__ void k_fill(float* p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

cudaError_t launch_fill(float* p, int64_t n, float v, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    k_fill<<<(unsigned)(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

// Eq. (7) confidence: the two planes the DTF turns into local moments.  The
// target is shifted by t[0] first: DT is row-stochastic, so V(t - k) = V(t) exactly, and
// the shift keeps DT(t^2) - DT(t)^2 from cancelling catastrophically in fp32 when |t| is
// large against its range (reading R22).
// Planes [t - t_0 ; (t - t_0)^2] and the epilogue, one thread per 4 consecutive pixels
// of a row: float4 on the pitched planes, and on the H x W target / outputs when W % 4 == 0
// (every row 16-B aligned); scalar otherwise
__global__ void __launch_bounds__(256) k_conf_prologue(const float* __restrict__ t, Geometry g, float* __restrict__ X) {
    const float k0 = __ldg(t);
    const int64_t per_row = g.pitch / 4;
    const int64_t n = g.H * per_row;
    const bool vec = (g.W & 3) == 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_row;
        const int64_t c = (i - r * per_row) * 4;
        if (c >= g.W) continue;
        float v[4];
        if (vec) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(t + r * g.W + c));
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = c + u < g.W ? __ldg(t + r * g.W + c + u) : k0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] -= k0;
        *reinterpret_cast<float4*>(X + r * g.pitch + c) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(X + g.plane + r * g.pitch + c) =
            make_float4(v[0] * v[0], v[1] * v[1], v[2] * v[2], v[3] * v[3]);
    }
}

__global__ void __launch_bounds__(256) k_conf_epilogue(const float* __restrict__ X, Geometry g, float inv_2sc2,
                                                       float* __restrict__ conf, float* __restrict__ var) {
    const int64_t per_row = g.pitch / 4;
    const int64_t n = g.H * per_row;
    const bool vec = (g.W & 3) == 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_row;
        const int64_t c = (i - r * per_row) * 4;
        if (c >= g.W) continue;
        const float4 a = __ldg(reinterpret_cast<const float4*>(X + r * g.pitch + c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(X + g.plane + r * g.pitch + c));
        const float m1[4] = {a.x, a.y, a.z, a.w}, m2[4] = {b.x, b.y, b.z, b.w};
        float v[4], e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v[u] = fmaxf(fmaf(-m1[u], m1[u], m2[u]), 0.f);  // DT(t^2) - DT(t)^2, clamped (R22)
            e[u] = __expf(-v[u] * inv_2sc2);
        }
        if (vec) {
            *reinterpret_cast<float4*>(conf + r * g.W + c) = make_float4(e[0], e[1], e[2], e[3]);
            if (var) *reinterpret_cast<float4*>(var + r * g.W + c) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c + u < g.W) {
                    conf[r * g.W + c + u] = e[u];
                    if (var) var[r * g.W + c + u] = v[u];
                }
        }
    }
}

static unsigned conf_blocks(const Geometry& g) {
    const int64_t n = g.H * (g.pitch / 4);
    const int64_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 16 ? b : 148 * 16);
}

cudaError_t launch_conf_prologue(const float* target, const Geometry& g, float* X, cudaStream_t s) {
    k_conf_prologue<<<conf_blocks(g), 256, 0, s>>>(target, g, X);
    return cudaGetLastError();
}

cudaError_t launch_conf_epilogue(const float* X, const Geometry& g, float inv_2sc2, float* conf, float* var,
                                 cudaStream_t s) {
    k_conf_epilogue<<<conf_blocks(g), 256, 0, s>>>(X, g, inv_2sc2, conf, var);
    return cudaGetLastError();
}

// Eq. (10) stereo step (R23), one-channel disparity z:
//     g = lam (z - zbar) + chat rho'(z - t) + gamma sum_k (I_L,k(x) - I_R,k(u)) dI_R,k/dx(u)
//     rho'(r) = r / sqrt(r^2 + eps^2),  u = x - z,  I_R linear along the row, clamped; slope 0 outside
// 2-D grid: blockIdx.y walks rows, threads columns; left / right are H x W x Cg HWC.
template <int CG>
__global__ void __launch_bounds__(256) k_update_stereo(const float* __restrict__ X, float* __restrict__ Z,
                                                       const float* __restrict__ T, const float* __restrict__ chat,
                                                       const float* __restrict__ left,
                                                       const float* __restrict__ right, int Cgr, Geometry g,
                                                       float lam, float step, float gamma, float eps,
                                                       float* __restrict__ out) {
    pdl_wait();
    const int Cg = CG > 0 ? CG : Cgr;
    const float e2 = eps * eps;
    for (int64_t r = blockIdx.y; r < g.H; r += gridDim.y) {
        const float* Lrow = left + r * g.W * Cg;
        const float* Rrow = right + r * g.W * Cg;
        for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.W; x += (int64_t)gridDim.x * blockDim.x) {
            const int64_t o = r * g.pitch + x;
            const float z = Z[o], zb = __ldg(X + o), t = __ldg(T + o), ch = __ldg(chat + o);
            const float res = z - t;
            const float rho1 = res * rsqrtf(fmaf(res, res, e2));  // Charbonnier derivative
            float gp = 0.f;
            if (gamma != 0.f && g.W > 1) {
                const float u = (float)x - z;
                const bool inside = u >= 0.f && u <= (float)(g.W - 1);
                const float uc = fminf(fmaxf(u, 0.f), (float)(g.W - 1));
                int64_t x0 = (int64_t)floorf(uc);
                if (x0 > g.W - 2) x0 = g.W - 2;
                const float f = uc - (float)x0;
                const float* ra = Rrow + x0 * Cg;
                const float* lp = Lrow + x * Cg;
                for (int k = 0; k < Cg; ++k) {
                    const float a = __ldg(ra + k), b = __ldg(ra + Cg + k);
                    const float iv = fmaf(f, b - a, a);
                    gp = fmaf(__ldg(lp + k) - iv, inside ? (b - a) : 0.f, gp);
                }
            }
            const float gr = fmaf(lam, z - zb, fmaf(ch, rho1, gamma * gp));
            const float zn = fmaf(-step, gr, z);
            if (out) out[r * g.W + x] = zn;
            else Z[o] = zn;
        }
    }
}

cudaError_t launch_update_stereo(const float* X, float* Z, const float* T, const float* chat, const float* left,
                                 const float* right, int Cg, const Geometry& g, float lam, float step, float gamma,
                                 float eps, float* out, cudaStream_t s) {
    const int64_t bx = (g.W + 255) / 256;
    dim3 grid((unsigned)(bx < 64 ? bx : 64), (unsigned)(g.H < 8192 ? g.H : 8192), 1);
    switch (Cg) {
        case 1:
            return launch_pdl(k_update_stereo<1>, grid, dim3(256), 0, s, X, Z, T, chat, left, right, Cg, g, lam, step,
                              gamma, eps, out);
        case 3:
            return launch_pdl(k_update_stereo<3>, grid, dim3(256), 0, s, X, Z, T, chat, left, right, Cg, g, lam, step,
                              gamma, eps, out);
        default:
            return launch_pdl(k_update_stereo<0>, grid, dim3(256), 0, s, X, Z, T, chat, left, right, Cg, g, lam, step,
                              gamma, eps, out);
    }
    return cudaGetLastError();
}

// Depth-SR front end (reading R24): bicubic (Catmull-Rom, a = -0.5) upsampling of
// the low-res depth by an integer factor f with clamped borders and centre alignment (high-res
// X reads low-res u = (X + 0.5)/f - 0.5), and the Gaussian-bump confidence
// exp(-dist^2 / (2 (f/4)^2)) around the nearest low-res sample centre.
__device__ __forceinline__ float cr_weight(float t) {
    t = fabsf(t);
    if (t < 1.f) return fmaf(t * t, fmaf(1.5f, t, -2.5f), 1.f);
    if (t < 2.f) return fmaf(t, fmaf(t, fmaf(-0.5f, t, 2.5f), -4.f), 2.f);
    return 0.f;
}

__global__ void __launch_bounds__(256) k_sr_prepare(const float* __restrict__ low, int64_t h, int64_t w, int f,
                                                    float* __restrict__ target, float* __restrict__ conf) {
    const int64_t H = h * f, W = w * f;
    const float inv = 1.f / (float)f, half = 0.5f * (float)(f - 1);
    const float k2 = 8.f / ((float)f * (float)f);  // 1 / (2 sigma_b^2), sigma_b = f / 4
    for (int64_t Y = blockIdx.y; Y < H; Y += gridDim.y) {
        const float v = ((float)Y + 0.5f) * inv - 0.5f;
        const int64_t j0 = (int64_t)floorf(v);
        float wy[4];
        int64_t jr[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int64_t j = j0 - 1 + d;
            wy[d] = cr_weight(v - (float)j);
            jr[d] = (j < 0 ? 0 : (j > h - 1 ? h - 1 : j)) * w;
        }
        int64_t kv = (int64_t)floorf(v + 0.5f);
        kv = kv < 0 ? 0 : (kv > h - 1 ? h - 1 : kv);
        const float dy = (float)Y - ((float)kv * (float)f + half);
        for (int64_t X = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; X < W; X += (int64_t)gridDim.x * blockDim.x) {
            const float u = ((float)X + 0.5f) * inv - 0.5f;
            const int64_t i0 = (int64_t)floorf(u);
            float acc = 0.f;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                int64_t i = i0 - 1 + d;
                const float wx = cr_weight(u - (float)i);
                i = i < 0 ? 0 : (i > w - 1 ? w - 1 : i);
                float col = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) col = fmaf(wy[e], __ldg(low + jr[e] + i), col);
                acc = fmaf(wx, col, acc);
            }
            int64_t ku = (int64_t)floorf(u + 0.5f);
            ku = ku < 0 ? 0 : (ku > w - 1 ? w - 1 : ku);
            const float dx = (float)X - ((float)ku * (float)f + half);
            target[Y * W + X] = acc;
            conf[Y * W + X] = __expf(-(dx * dx + dy * dy) * k2);
        }
    }
}

cudaError_t launch_sr_prepare(const float* low, int64_t h, int64_t w, int f, float* target, float* conf,
                              cudaStream_t s) {
    const int64_t H = h * f, W = w * f;
    const int64_t bx = (W + 255) / 256;
    dim3 grid((unsigned)(bx < 64 ? bx : 64), (unsigned)(H < 8192 ? H : 8192), 1);
    k_sr_prepare<<<grid, 256, 0, s>>>(low, h, w, f, target, conf);
    return cudaGetLastError();
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is per function AND per device: remember, per
// (device, function), the largest value set so far, under a lock (one process may drive
// several GPUs from several threads)
cudaError_t ensure_smem_attr(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, const void*>, size_t>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& en : done)
        if (en.first.first == dev && en.first.second == fn) {
            if (en.second >= bytes) return cudaSuccess;
            if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) != cudaSuccess)
                return e;
            en.second = bytes;
            return cudaSuccess;
        }
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) != cudaSuccess)
        return e;
    done.push_back({{dev, fn}, bytes});
    return cudaSuccess;
}

}  // namespace dts
