// k_col.cu -- K3/K4: one recursive-filter pass along every column (sm_100a),
// optionally fused with the solver update of Eq. (3).
//
// Same recurrence as K2 along columns (top->bottom causal, bottom->top anticausal)
// with A = a_i^{d_y} (R4-R6).  MODE_UPDATE fuses the DTS gradient
// step into the write-out of the last column pass:
//     zbar = column-pass output;   z <- z - step * [lambda (z - zbar) + chat (z - t)]
// MODE_SUPPORT multiplies the two-sided unnormalised column sums s_y into S (R7).
//
// Design: one thread per column -- a warp covers 32 adjacent
// columns, so every access of a warp is one 128-B row segment.  A column tile
// (32 columns x H rows) is held ON CHIP by a thread-block cluster of CB CTAs (CTA b
// holds rows [b*HB, (b+1)*HB) in shared memory), so each pixel is read from HBM
// once and written once per pass:
//   1. TMA (cp.async.bulk.tensor) streams the band in, one box and one mbarrier per
//      segment of Ls rows, so warp s starts folding as soon as its rows land;
//   2. each thread folds its Ls rows into an affine map; the S maps of a column
//      are scanned by a warp-shuffle scan (lane = segment);
//   3. per-band totals are exchanged between the cluster's CTAs through
//      distributed shared memory (DSMEM): causal carries, then anticausal carries;
//   4. the band is re-swept with exact carries in shared memory and leaves by TMA
//      tensor stores (FILTER) or a vectorised, fully parallel update loop (UPDATE).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dts_device.cuh"
#include "dts_launch.h"

namespace dts {

constexpr int TW = 32;  // columns per tile (one warp)

struct ColParams {
    float* x;        // planar state (FILTER/UPDATE input; FILTER output through tm_x)
    const float* d;  // d_y (halo row)
    float* support;  // SUPPORT: S, multiplied in place by s_y
    UpdateArgs upd;
    int64_t plane, pitch;
    int H, W, HB, S, Ls, CB;
    float kc;
};

struct ColSmem {  // float offsets into dynamic shared memory
    int xs, As, segC, segA, tot, rem, carry, bars;
    size_t bytes;
};

__host__ __device__ inline ColSmem col_smem_layout(int NV, bool hasx, int HB, int S, int CB) {
    ColSmem L;
    int o = 0;
    L.xs = o;
    o += NV * HB * TW;  // samples / y / zbar (SUPPORT: P, then s_y)
    (void)hasx;
    L.As = o;
    o += (HB + 1) * TW;  // + halo row
    L.segC = o;
    o += (NV + 1) * S * (TW + 1);
    L.segA = o;
    o += (NV + 1) * S * (TW + 1);
    L.tot = o;  // [2][NV+1][TW]: causal, anticausal band totals (read remotely)
    o += 2 * (NV + 1) * TW;
    L.rem = o;  // gathered remote totals [CB][NV+1][TW]
    o += CB * (NV + 1) * TW;
    L.carry = o;  // [NV][TW]
    o += NV * TW;
    o = (o + 1) & ~1;  // 8-B alignment for the mbarriers
    L.bars = o;
    o += 2 * S;
    L.bytes = (size_t)o * sizeof(float);
    return L;
}

// Warp-shuffle scan across the S segment maps of column `cc` (lane = segment).
// Forward: exclusive prefix (composite of segments < lane), written back in place.
// Reverse: exclusive suffix (composite of segments > lane, applied right to left).
// Lanes >= S act as identity.  Returns the total (valid in every lane).
template <int NV, bool REV>
__device__ __forceinline__ void seg_scan(float* seg, int S, int cc, float* tot) {
    const int lane = threadIdx.x & 31;
    Aff<NV> v = aff_identity<NV>();
    if (lane < S) {
        v.P = seg[(0 * S + lane) * (TW + 1) + cc];
#pragma unroll
        for (int k = 0; k < NV; ++k) v.B[k] = seg[((1 + k) * S + lane) * (TW + 1) + cc];
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Aff<NV> e;
        e.P = REV ? __shfl_down_sync(FULL, v.P, off) : __shfl_up_sync(FULL, v.P, off);
#pragma unroll
        for (int k = 0; k < NV; ++k) e.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], off) : __shfl_up_sync(FULL, v.B[k], off);
        const bool take = REV ? (lane + off < 32) : (lane >= off);
        if (take) v = aff_compose(e, v);
    }
    Aff<NV> ex;
    ex.P = REV ? __shfl_down_sync(FULL, v.P, 1) : __shfl_up_sync(FULL, v.P, 1);
#pragma unroll
    for (int k = 0; k < NV; ++k) ex.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], 1) : __shfl_up_sync(FULL, v.B[k], 1);
    if (REV ? lane == 31 : lane == 0) ex = aff_identity<NV>();
    // total = inclusive value at the last position in scan order
    const int src = REV ? 0 : 31;
    Aff<NV> t;
    t.P = __shfl_sync(FULL, v.P, src);
#pragma unroll
    for (int k = 0; k < NV; ++k) t.B[k] = __shfl_sync(FULL, v.B[k], src);
    if (lane < S) {
        seg[(0 * S + lane) * (TW + 1) + cc] = ex.P;
#pragma unroll
        for (int k = 0; k < NV; ++k) seg[((1 + k) * S + lane) * (TW + 1) + cc] = ex.B[k];
    }
    if (lane == 0) {
        tot[0 * TW + cc] = t.P;
#pragma unroll
        for (int k = 0; k < NV; ++k) tot[(1 + k) * TW + cc] = t.B[k];
    }
}

template <int CT, int MODE>
__global__ void __launch_bounds__(1024, 1)
    k_col_pass(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_d, const ColParams p) {
    constexpr int NV = (MODE == MODE_SUPPORT) ? 1 : CT;
    constexpr bool HASX = MODE != MODE_SUPPORT;
    extern __shared__ __align__(128) float smem[];
    const int HB = p.HB, S = p.S, Ls = p.Ls, CB = p.CB;
    const ColSmem L = col_smem_layout(NV, HASX, HB, S, CB);
    float* xs = smem + L.xs;
    float* As = smem + L.As;
    float* segC = smem + L.segC;
    float* segA = smem + L.segA;
    float* totC = smem + L.tot;
    float* totA = smem + L.tot + (NV + 1) * TW;
    float* rem = smem + L.rem;
    float* carry = smem + L.carry;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);

    const int c = threadIdx.x & 31;
    const int s = threadIdx.x >> 5;  // segment == warp
    const int col0 = blockIdx.x * TW;
    const int col = col0 + c;
    const bool colok = col < p.W;
    const int band = (CB > 1) ? (int)cluster_ctarank() : 0;
    const int r0 = band * HB;

    // ---- 1. TMA: one box per segment and array, one mbarrier per segment ----
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tm_d);
        if (HASX) tma_prefetch_desc(&tm_x);
        const uint32_t box = (uint32_t)(Ls * TW * sizeof(float));
        for (int q = 0; q < S; ++q) {
            const int rq = r0 + q * Ls;
            const uint32_t bytes = rq < p.H ? box * (1 + (HASX ? NV : 0)) : 0u;
            mbar_arrive_expect_tx(&bars[q], bytes);
            if (bytes) {
                tma_load_2d(As + q * Ls * TW, &tm_d, col0, rq, &bars[q]);
                if constexpr (HASX) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) tma_load_3d(xs + (v * HB + q * Ls) * TW, &tm_x, col0, rq, v, &bars[q]);
                }
            }
        }
    }
    if (s == 0) {  // halo: coefficient of the first row of the next band
        const int rh = r0 + HB;
        As[HB * TW + c] = (colok && rh < p.H) ? coef_from_d(p.d[(int64_t)rh * p.pitch + col], p.kc) : 0.f;
    }

    // ---- 2. causal fold (d -> A in place, invalid samples zeroed) ----
    const int lo = s * Ls;
    mbar_wait(&bars[s], 0);
    Aff<NV> m = aff_identity<NV>();
    for (int j = 0; j < Ls; ++j) {
        const int rr = lo + j;
        const bool ok = colok && (r0 + rr) < p.H;
        const float a = ok ? coef_from_d(As[rr * TW + c], p.kc) : 0.f;
        As[rr * TW + c] = a;
        m.P *= a;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if constexpr (HASX) {
                float* px = xs + (v * HB + rr) * TW + c;
                const float xv = ok ? *px : 0.f;
                *px = xv;
                m.B[v] = fmaf(a, m.B[v] - xv, xv);
            } else {
                m.B[v] = fmaf(a, m.B[v], 1.f);
            }
        }
    }
    segC[(0 * S + s) * (TW + 1) + c] = m.P;
#pragma unroll
    for (int v = 0; v < NV; ++v) segC[((1 + v) * S + s) * (TW + 1) + c] = m.B[v];
    __syncthreads();
    for (int cc = s; cc < TW; cc += S) seg_scan<NV, false>(segC, S, cc, totC);
    if (CB > 1) cluster_sync_all(); else __syncthreads();

    // ---- 3a. causal carry into the band: compose the totals of the bands above ----
    for (int q = s; q < band; q += S) {
#pragma unroll
        for (int k = 0; k < NV + 1; ++k) rem[(q * (NV + 1) + k) * TW + c] = ld_dsmem_f32(totC + k * TW + c, q);
    }
    __syncthreads();
    if (s == 0) {
        float cin[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) cin[v] = 0.f;
        for (int q = 0; q < band; ++q) {
            const float P = rem[(q * (NV + 1)) * TW + c];
#pragma unroll
            for (int v = 0; v < NV; ++v) cin[v] = fmaf(P, cin[v], rem[(q * (NV + 1) + 1 + v) * TW + c]);
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) carry[v * TW + c] = cin[v];
    }
    __syncthreads();

    // ---- 4. causal apply (y -> xs) + forward accumulation of the anticausal map ----
    // z[n] = a z[n+1] + b_n, a = A[n+1], b_n = (1 - a) y[n] (filter) or 1 (support);
    // segment map z_lo = Q z_hi + E accumulated forward: E += Q b_n; Q *= a.
    {
        float y[NV];
        const float eP = segC[(0 * S + s) * (TW + 1) + c];
#pragma unroll
        for (int v = 0; v < NV; ++v) y[v] = fmaf(eP, carry[v * TW + c], segC[((1 + v) * S + s) * (TW + 1) + c]);
        Aff<NV> am = aff_identity<NV>();
        for (int j = 0; j < Ls; ++j) {
            const int rr = lo + j;
            const float a = As[rr * TW + c];
            const float an = As[(rr + 1) * TW + c];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                float* px = xs + (v * HB + rr) * TW + c;
                if constexpr (HASX) {
                    const float xv = *px;
                    y[v] = fmaf(a, y[v] - xv, xv);
                    am.B[v] = fmaf(am.P * (1.f - an), y[v], am.B[v]);
                } else {
                    y[v] = fmaf(a, y[v], 1.f);
                    am.B[v] += am.P;
                }
                *px = y[v];
            }
            am.P *= an;
        }
        segA[(0 * S + s) * (TW + 1) + c] = am.P;
#pragma unroll
        for (int v = 0; v < NV; ++v) segA[((1 + v) * S + s) * (TW + 1) + c] = am.B[v];
    }
    __syncthreads();
    for (int cc = s; cc < TW; cc += S) seg_scan<NV, true>(segA, S, cc, totA);
    if (CB > 1) cluster_sync_all(); else __syncthreads();

    // ---- 5. anticausal carry from the bands below ----
    for (int q = band + 1 + s; q < CB; q += S) {
#pragma unroll
        for (int k = 0; k < NV + 1; ++k) rem[(q * (NV + 1) + k) * TW + c] = ld_dsmem_f32(totA + k * TW + c, q);
    }
    if (CB > 1) cluster_arrive();  // this CTA's remote reads are issued and consumed above
    __syncthreads();
    if (s == 0) {
        float ein[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) ein[v] = 0.f;
        for (int q = CB - 1; q > band; --q) {
            const float Q = rem[(q * (NV + 1)) * TW + c];
#pragma unroll
            for (int v = 0; v < NV; ++v) ein[v] = fmaf(Q, ein[v], rem[(q * (NV + 1) + 1 + v) * TW + c]);
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) carry[v * TW + c] = ein[v];
    }
    __syncthreads();

    // ---- 6. anticausal apply (bottom -> top), zbar (or s_y) back into xs ----
    {
        float z[NV];
        const float eQ = segA[(0 * S + s) * (TW + 1) + c];
#pragma unroll
        for (int v = 0; v < NV; ++v) z[v] = fmaf(eQ, carry[v * TW + c], segA[((1 + v) * S + s) * (TW + 1) + c]);
        for (int j = Ls - 1; j >= 0; --j) {
            const int rr = lo + j;
            const float an = As[(rr + 1) * TW + c];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                float* px = xs + (v * HB + rr) * TW + c;
                const float yv = *px;
                if constexpr (HASX) {
                    z[v] = fmaf(an, z[v] - yv, yv);
                    *px = z[v];
                } else {
                    z[v] = fmaf(an, z[v], 1.f);
                    *px = yv + z[v] - 1.f;  // s_y = P + Q - 1
                }
            }
        }
    }

    // ---- 7. write-out ----
    const int nrows = max(0, min(HB, p.H - r0));
    if constexpr (MODE == MODE_FILTER) {
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < S; ++q) {
                const int rq = r0 + q * Ls;
                if (rq >= p.H) break;
#pragma unroll
                for (int v = 0; v < NV; ++v) tma_store_3d(&tm_x, col0, rq, v, xs + (v * HB + q * Ls) * TW);
            }
            bulk_commit();
            bulk_wait_read0();
        }
    } else {
        __syncthreads();
        const int nitems = nrows * (TW / 4);
#pragma unroll 4
        for (int i = threadIdx.x; i < nitems; i += blockDim.x) {
            const int rr = i >> 3;
            const int q4 = (i & 7) * 4;
            const int64_t r = r0 + rr;
            const int cq = col0 + q4;
            if constexpr (MODE == MODE_SUPPORT) {
                const float4 sy = *reinterpret_cast<const float4*>(xs + rr * TW + q4);
                float4* ps = reinterpret_cast<float4*>(p.support + r * p.pitch + cq);
                float4 sv = *ps;
                sv.x *= sy.x;
                sv.y *= sy.y;
                sv.z *= sy.z;
                sv.w *= sy.w;
                *ps = sv;
            } else {
                const float4 ch = __ldg(reinterpret_cast<const float4*>(p.upd.chat + r * p.pitch + cq));
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int64_t idx = v * p.plane + r * p.pitch + cq;
                    const float4 zb = *reinterpret_cast<const float4*>(xs + (v * HB + rr) * TW + q4);
                    const float4 zo = *reinterpret_cast<const float4*>(p.upd.Z + idx);
                    const float4 tv = __ldg(reinterpret_cast<const float4*>(p.upd.T + idx));
                    float4 zn;
                    zn.x = fmaf(-p.upd.step, fmaf(p.upd.lam, zo.x - zb.x, ch.x * (zo.x - tv.x)), zo.x);
                    zn.y = fmaf(-p.upd.step, fmaf(p.upd.lam, zo.y - zb.y, ch.y * (zo.y - tv.y)), zo.y);
                    zn.z = fmaf(-p.upd.step, fmaf(p.upd.lam, zo.z - zb.z, ch.z * (zo.z - tv.z)), zo.z);
                    zn.w = fmaf(-p.upd.step, fmaf(p.upd.lam, zo.w - zb.w, ch.w * (zo.w - tv.w)), zo.w);
                    if (p.upd.out_hwc) {
                        const float zz[4] = {zn.x, zn.y, zn.z, zn.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (cq + u < p.W) p.upd.out_hwc[(r * p.W + cq + u) * CT + v] = zz[u];
                    } else {
                        *reinterpret_cast<float4*>(p.upd.Z + idx) = zn;
                    }
                }
            }
        }
    }
    if (CB > 1) cluster_wait();  // keep shared memory alive until every CTA finished reading it
}

// ---------------------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// rank-3 map over planar fp32 data [planes][H][pitch] with box {TW, rows, 1}
static bool make_tmap(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int64_t planes, int rows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)H, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * sizeof(float)), (cuuint64_t)(pitch * H * sizeof(float))};
    cuuint32_t box[3] = {(cuuint32_t)TW, (cuuint32_t)rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
static bool make_tmap2(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int rows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)H};
    cuuint64_t strides[1] = {(cuuint64_t)(pitch * sizeof(float))};
    cuuint32_t box[2] = {(cuuint32_t)TW, (cuuint32_t)rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static const size_t kSmemMax = 227 * 1024;

cudaError_t plan_col_pass(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan) {
    (void)num_sms;
    const int NV = (mode == MODE_SUPPORT) ? 1 : Ct;
    const bool hasx = mode != MODE_SUPPORT;
    for (int CB = 1; CB <= 16; CB *= 2) {
        const int64_t HBmin = (g.H + CB - 1) / CB;
        int S = (int)((HBmin + 31) / 32);
        S = S < 1 ? 1 : (S > 32 ? 32 : S);
        const int Ls = (int)((HBmin + S - 1) / S);
        if (Ls > 256) continue;  // TMA box limit
        S = (int)((HBmin + Ls - 1) / Ls);
        const int HB = S * Ls;
        const ColSmem L = col_smem_layout(NV, hasx, HB, S, CB);
        if (L.bytes > kSmemMax) continue;
        plan->TW = TW;
        plan->CB = CB;
        plan->HB = HB;
        plan->S = S;
        plan->Ls = Ls;
        plan->threads = TW * S;
        plan->grid = dim3((unsigned)((g.W + TW - 1) / TW), (unsigned)CB, 1);
        plan->smem = L.bytes;
        return cudaSuccess;
    }
    return cudaErrorInvalidValue;
}

template <int CT, int MODE>
static cudaError_t launch_t(const ColPlan& plan, const CUtensorMap& tx, const CUtensorMap& td, const ColParams& p,
                            cudaStream_t s) {
    static size_t configured = 0;
    static bool nonportable = false;
    auto fn = k_col_pass<CT, MODE>;
    if (plan.smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
        if (e != cudaSuccess) return e;
        configured = plan.smem;
    }
    if (plan.CB > 8 && !nonportable) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        nonportable = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = plan.grid;
    cfg.blockDim = dim3((unsigned)plan.threads, 1, 1);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = (unsigned)plan.CB;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, tx, td, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_ct(const ColPlan& plan, const CUtensorMap& tx, const CUtensorMap& td, const ColParams& p,
                             int Ct, cudaStream_t s) {
    switch (Ct) {
        case 1: return launch_t<1, MODE>(plan, tx, td, p, s);
        case 2: return launch_t<2, MODE>(plan, tx, td, p, s);
        case 3: return launch_t<3, MODE>(plan, tx, td, p, s);
        case 4: return launch_t<4, MODE>(plan, tx, td, p, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_col_pass(const ColPlan& plan, const Geometry& g, int Ct, int mode, float* x, const float* d,
                            float kc, const UpdateArgs* upd, float* support, cudaStream_t s) {
    ColParams p = {};
    p.x = x;
    p.d = d;
    p.support = support;
    if (upd) p.upd = *upd;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.HB = plan.HB;
    p.S = plan.S;
    p.Ls = plan.Ls;
    p.CB = plan.CB;
    p.kc = kc;
    CUtensorMap tx, td;
    if (!make_tmap2(&td, d, g.pitch, g.H, plan.Ls)) return cudaErrorInvalidValue;
    if (mode != MODE_SUPPORT) {
        if (!make_tmap(&tx, x, g.pitch, g.H, Ct, plan.Ls)) return cudaErrorInvalidValue;
    } else {
        tx = td;  // unused
    }
    switch (mode) {
        case MODE_FILTER: return launch_ct<MODE_FILTER>(plan, tx, td, p, Ct, s);
        case MODE_UPDATE: return launch_ct<MODE_UPDATE>(plan, tx, td, p, Ct, s);
        case MODE_SUPPORT: return launch_t<1, MODE_SUPPORT>(plan, tx, td, p, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace dts
