// k_col.cu -- K3/K4: one recursive-filter pass along every column (sm_100a),
// optionally fused with the solver update of Eq. (3).
//
// Same recurrence as K2 along columns (top->bottom causal, bottom->top anticausal)
// with A = a_i^{d_y} (R4-R6).  MODE_UPDATE fuses the DTS gradient
// step into the anticausal sweep of the last column pass:
//     zbar = column-pass output;   z <- z - step * [lambda (z - zbar) + chat (z - t)]
// MODE_SUPPORT multiplies the two-sided unnormalised column sums s_y into S (R7).
//
// Design: one thread per column -- a warp covers 32 adjacent
// columns, so every global access of a warp is one 128-B row segment.  A column
// tile (TW columns x H rows) is held ON CHIP by a thread-block cluster of CB CTAs
// (CTA b holds rows [b*HB, (b+1)*HB) of the tile in shared memory), so each pixel
// is read from HBM once and written once per pass.  Inside a CTA each thread owns
// Ls consecutive rows of one column ("segment"); the per-segment affine maps are
// combined serially per column in shared memory, and the per-band totals are
// exchanged between the CTAs of the cluster through distributed shared memory
// (DSMEM).  Two exchanges per pass: causal carries, then anticausal carries.
#include "dts_device.cuh"
#include "dts_launch.h"

namespace dts {

struct ColParams {
    float* x;            // planar state (FILTER/UPDATE: in; FILTER: out, in place)
    const float* d;      // d_y
    float* support;      // SUPPORT: S, multiplied in place by s_y
    UpdateArgs upd;
    int64_t plane, pitch;
    int H, W, HB, S, Ls, CB;
    float kc;
};

template <int TW, int CT, int MODE>
__global__ void __launch_bounds__(1024) k_col_pass(const ColParams p) {
    constexpr int NV = (MODE == MODE_SUPPORT) ? 1 : CT;
    extern __shared__ __align__(128) float smem[];
    // layout: xs[NV][HB][TW] | As[HB+1][TW] | segC[S][TW][NV+1] | segA[S][TW][NV+1] |
    //         totC[TW][NV+1] | totA[TW][NV+1] | carry[TW][NV]
    const int HB = p.HB, S = p.S, Ls = p.Ls;
    float* xs = smem;
    float* As = xs + (int64_t)NV * HB * TW;
    float* segC = As + (int64_t)(HB + 1) * TW;
    float* segA = segC + S * TW * (NV + 1);
    float* totC = segA + S * TW * (NV + 1);
    float* totA = totC + TW * (NV + 1);
    float* carry = totA + TW * (NV + 1);

    const int c = threadIdx.x % TW;
    const int s = threadIdx.x / TW;
    const int col = blockIdx.x * TW + c;
    const bool colok = col < p.W;
    const int band = (p.CB > 1) ? (int)cluster_ctarank() : 0;
    const int r0 = band * HB;
    const int nrows = max(0, min(HB, p.H - r0));  // valid rows of this band

    // ---- 1. stage the band tile: samples and coefficients (masked) ----
    for (int rr = s; rr <= HB; rr += S) {
        const int64_t r = (int64_t)r0 + rr;
        const bool ok = colok && r < p.H;
        if (rr < HB) {
            if constexpr (MODE != MODE_SUPPORT) {
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    xs[((int64_t)v * HB + rr) * TW + c] = ok ? p.x[v * p.plane + r * p.pitch + col] : 0.f;
            }
        }
        As[rr * TW + c] = ok ? coef_from_d(p.d[r * p.pitch + col], p.kc) : 0.f;  // rr == HB: halo row
    }
    __syncthreads();

    const int lo = s * Ls;
    const int hi = min(lo + Ls, HB);

    // ---- 2. causal fold of this thread's segment ----
    Aff<NV> m = aff_identity<NV>();
    for (int rr = lo; rr < hi; ++rr) {
        const float a = As[rr * TW + c];
        m.P *= a;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if constexpr (MODE == MODE_SUPPORT) m.B[v] = fmaf(a, m.B[v], 1.f);
            else {
                const float xv = xs[((int64_t)v * HB + rr) * TW + c];
                m.B[v] = fmaf(a, m.B[v] - xv, xv);
            }
        }
    }
    {
        float* e = segC + (s * TW + c) * (NV + 1);
        e[0] = m.P;
#pragma unroll
        for (int v = 0; v < NV; ++v) e[1 + v] = m.B[v];
    }
    __syncthreads();
    // ---- 3. in-CTA segment scan per column (exclusive, written back), band total ----
    if (s == 0) {
        Aff<NV> run = aff_identity<NV>();
        for (int q = 0; q < S; ++q) {
            float* e = segC + (q * TW + c) * (NV + 1);
            Aff<NV> cur;
            cur.P = e[0];
#pragma unroll
            for (int v = 0; v < NV; ++v) cur.B[v] = e[1 + v];
            e[0] = run.P;
#pragma unroll
            for (int v = 0; v < NV; ++v) e[1 + v] = run.B[v];
            run = aff_compose(run, cur);
        }
        float* tt = totC + c * (NV + 1);
        tt[0] = run.P;
#pragma unroll
        for (int v = 0; v < NV; ++v) tt[1 + v] = run.B[v];
    }
    if (p.CB > 1) cluster_sync_all(); else __syncthreads();
    // ---- 4. causal carry into the band from the bands above (DSMEM) ----
    if (s == 0) {
        float cin[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) cin[v] = 0.f;
        for (int bb = 0; bb < band; ++bb) {
            const float P = ld_dsmem_f32(totC + c * (NV + 1), bb);
#pragma unroll
            for (int v = 0; v < NV; ++v) cin[v] = fmaf(P, cin[v], ld_dsmem_f32(totC + c * (NV + 1) + 1 + v, bb));
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) carry[c * NV + v] = cin[v];
    }
    __syncthreads();

    // ---- 5. causal apply (y into xs) + forward accumulation of the anticausal map ----
    // anticausal step for row n: z[n] = a z[n+1] + b_n with a = A[n+1],
    // b_n = (1 - a) y[n] (filter) or 1 (support); the segment map z_lo = Q z_hi + E
    // is accumulated in forward order: E += Q * b_n; Q *= a.
    Aff<NV> am = aff_identity<NV>();
    {
        const float* e = segC + (s * TW + c) * (NV + 1);
        float y[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) y[v] = fmaf(e[0], carry[c * NV + v], e[1 + v]);
        for (int rr = lo; rr < hi; ++rr) {
            const float a = As[rr * TW + c];
            const float an = As[(rr + 1) * TW + c];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                float* px = xs + ((int64_t)v * HB + rr) * TW + c;
                if constexpr (MODE == MODE_SUPPORT) {
                    y[v] = fmaf(a, y[v], 1.f);
                    am.B[v] = fmaf(am.P, 1.f, am.B[v]);
                } else {
                    y[v] = fmaf(a, y[v] - *px, *px);
                    am.B[v] = fmaf(am.P * (1.f - an), y[v], am.B[v]);
                }
                *px = y[v];
            }
            am.P *= an;
        }
    }
    {
        float* e = segA + (s * TW + c) * (NV + 1);
        e[0] = am.P;
#pragma unroll
        for (int v = 0; v < NV; ++v) e[1 + v] = am.B[v];
    }
    __syncthreads();
    // ---- 6. reverse segment scan per column, band total, anticausal carry (DSMEM) ----
    if (s == 0) {
        Aff<NV> run = aff_identity<NV>();
        for (int q = S - 1; q >= 0; --q) {
            float* e = segA + (q * TW + c) * (NV + 1);
            Aff<NV> cur;
            cur.P = e[0];
#pragma unroll
            for (int v = 0; v < NV; ++v) cur.B[v] = e[1 + v];
            e[0] = run.P;
#pragma unroll
            for (int v = 0; v < NV; ++v) e[1 + v] = run.B[v];
            run = aff_compose(run, cur);
        }
        float* tt = totA + c * (NV + 1);
        tt[0] = run.P;
#pragma unroll
        for (int v = 0; v < NV; ++v) tt[1 + v] = run.B[v];
    }
    if (p.CB > 1) cluster_sync_all(); else __syncthreads();
    if (s == 0) {
        float ein[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) ein[v] = 0.f;
        for (int bb = p.CB - 1; bb > band; --bb) {
            const float Q = ld_dsmem_f32(totA + c * (NV + 1), bb);
#pragma unroll
            for (int v = 0; v < NV; ++v) ein[v] = fmaf(Q, ein[v], ld_dsmem_f32(totA + c * (NV + 1) + 1 + v, bb));
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) carry[c * NV + v] = ein[v];
    }
    if (p.CB > 1) cluster_arrive();  // this CTA's remote reads are done
    __syncthreads();

    // ---- 7. anticausal apply (bottom -> top) and output ----
    {
        const float* e = segA + (s * TW + c) * (NV + 1);
        float z[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) z[v] = fmaf(e[0], carry[c * NV + v], e[1 + v]);
        const int vhi = min(hi, nrows);
        for (int rr = hi - 1; rr >= lo; --rr) {
            const float an = As[(rr + 1) * TW + c];
            const int64_t r = (int64_t)r0 + rr;
            const bool ok = colok && rr < vhi;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float yv = xs[((int64_t)v * HB + rr) * TW + c];
                if constexpr (MODE == MODE_SUPPORT) {
                    z[v] = fmaf(an, z[v], 1.f);
                    if (ok) p.support[r * p.pitch + col] *= (yv + z[v] - 1.f);
                } else {
                    z[v] = fmaf(an, z[v] - yv, yv);
                    if (ok) {
                        if constexpr (MODE == MODE_FILTER) {
                            p.x[v * p.plane + r * p.pitch + col] = z[v];
                        } else {  // MODE_UPDATE: Eq. (3) step with zbar = z[v]
                            const int64_t idx = v * p.plane + r * p.pitch + col;
                            const float zo = p.upd.Z[idx];
                            const float tv = p.upd.T[idx];
                            const float ch = p.upd.chat[r * p.pitch + col];
                            const float g = fmaf(p.upd.lam, zo - z[v], ch * (zo - tv));
                            const float zn = fmaf(-p.upd.step, g, zo);
                            if (p.upd.out_hwc) p.upd.out_hwc[(r * p.W + col) * CT + v] = zn;
                            else p.upd.Z[idx] = zn;
                        }
                    }
                }
            }
        }
    }
    if (p.CB > 1) cluster_wait();  // keep shared memory alive until every CTA finished reading it
}

// ---------------------------------------------------------------------------------------

static size_t col_smem_bytes(int TW, int NV, int HB, int S) {
    return sizeof(float) * ((size_t)NV * HB * TW + (size_t)(HB + 1) * TW + 2 * (size_t)S * TW * (NV + 1) +
                            2 * (size_t)TW * (NV + 1) + (size_t)TW * NV);
}

cudaError_t plan_col_pass(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan) {
    (void)num_sms;
    const int NV = (mode == MODE_SUPPORT) ? 1 : Ct;
    const int TW = 32;
    const size_t budget = 200 * 1024;
    int CB = 1;
    int HB = 0, S = 0, Ls = 0;
    for (;; CB *= 2) {
        if (CB > 16) return cudaErrorInvalidValue;
        HB = (int)((g.H + CB - 1) / CB);
        S = (HB + 31) / 32;
        if (S < 1) S = 1;
        if (S > 32) S = 32;
        Ls = (HB + S - 1) / S;
        S = (HB + Ls - 1) / Ls;
        if (col_smem_bytes(TW, NV, HB, S) <= budget) break;
    }
    plan->TW = TW;
    plan->CB = CB;
    plan->HB = HB;
    plan->S = S;
    plan->Ls = Ls;
    plan->threads = TW * S;
    plan->grid = dim3((unsigned)((g.W + TW - 1) / TW), (unsigned)CB, 1);
    plan->smem = col_smem_bytes(TW, NV, HB, S);
    return cudaSuccess;
}

template <int CT, int MODE>
static cudaError_t launch_t(const ColPlan& plan, const ColParams& p, cudaStream_t s) {
    static size_t configured = 0;
    static bool nonportable = false;
    auto fn = k_col_pass<32, CT, MODE>;
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_ct(const ColPlan& plan, const ColParams& p, int Ct, cudaStream_t s) {
    switch (Ct) {
        case 1: return launch_t<1, MODE>(plan, p, s);
        case 2: return launch_t<2, MODE>(plan, p, s);
        case 3: return launch_t<3, MODE>(plan, p, s);
        case 4: return launch_t<4, MODE>(plan, p, s);
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
    switch (mode) {
        case MODE_FILTER: return launch_ct<MODE_FILTER>(plan, p, Ct, s);
        case MODE_UPDATE: return launch_ct<MODE_UPDATE>(plan, p, Ct, s);
        case MODE_SUPPORT: return launch_t<1, MODE_SUPPORT>(plan, p, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace dts
