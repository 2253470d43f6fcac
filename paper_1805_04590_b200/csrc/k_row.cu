// k_row.cu -- K2: one recursive-filter pass along every row (sm_100a).
//
// Computes, for each row of every channel plane, the domain-transform recursive
// filter of BASELINE.json's north star / DESIGN.md R4:
//     causal      y[0] = x[0],       y[k] = (1 - A[k]) x[k] + A[k] y[k-1]
//     anticausal  z[W-1] = y[W-1],   z[k] = (1 - A[k+1]) y[k] + A[k+1] z[k+1]
// with A[k] = a_i^{d_x[k]} = 2^(-kc d_x[k]) (R5), A = 0 at the +inf sentinel.
// SUPPORT mode computes the unnormalised two-sided sums of R7 instead:
//     P[k] = 1 + A[k] P[k-1],  Q[k] = 1 + A[k+1] Q[k+1],  s_x = P + Q - 1.
//
// Design: each row is one linear-recurrence scan.  A group of G
// threads owns a row; thread t keeps L consecutive samples in registers, folds
// them into an affine map, the G maps are combined by a shuffle (+ smem across
// warps) scan, and the thread re-applies its chunk with the exact carry -- causal
// and anticausal fused in one kernel, so a row is read once and written once.
// Rows are staged with TMA bulk copies (cp.async.bulk) into a double buffer by a
// persistent CTA: the next row group streams in while the current one computes,
// and results leave through bulk shared->global stores.
#include "dts_device.cuh"
#include "dts_launch.h"

namespace dts {

struct RowParams {
    const float* in;
    float* out;
    const float* d;
    // MODE_ROWUPD: Eq. (3) step applied on the fly, Z <- Z - step [lam (Z - in) + chat (Z - T)],
    // and the new Z is the row filter's input (in = zbar of the previous iteration)
    float* Z;
    const float* T;
    const float* chat;
    float lam, step;
    int64_t plane, pitch, rowstride;
    int64_t rowlen;  // floats staged per row (the pitch; a row strip's padded width)
    int pdl_early;   // trigger the dependent launch at the start (option pdl = 2) instead of the end
    int H, W, G, R, nbuf;
    float kc;
};

// Exclusive scan of affine maps over the G threads of a row group, in thread order
// (REV = false) or reverse thread order (REV = true).  Must be called by every
// thread of the CTA (contains __syncthreads when G > 32).
template <int NV, bool REV>
__device__ __forceinline__ Aff<NV> group_exclusive_scan(Aff<NV> v, int t, int G, float* scratch) {
    const int lane = threadIdx.x & 31;
    const int width = G < 32 ? G : 32;
    const int li = lane & (width - 1);
    const int pos = REV ? (width - 1 - li) : li;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= width) break;
        Aff<NV> e;
        e.P = REV ? __shfl_down_sync(FULL, v.P, off, width) : __shfl_up_sync(FULL, v.P, off, width);
#pragma unroll
        for (int c = 0; c < NV; ++c)
            e.B[c] = REV ? __shfl_down_sync(FULL, v.B[c], off, width) : __shfl_up_sync(FULL, v.B[c], off, width);
        if (pos >= off) v = aff_compose(e, v);
    }
    // inclusive -> exclusive within the warp segment
    Aff<NV> ex;
    ex.P = REV ? __shfl_down_sync(FULL, v.P, 1, width) : __shfl_up_sync(FULL, v.P, 1, width);
#pragma unroll
    for (int c = 0; c < NV; ++c)
        ex.B[c] = REV ? __shfl_down_sync(FULL, v.B[c], 1, width) : __shfl_up_sync(FULL, v.B[c], 1, width);
    if (pos == 0) ex = aff_identity<NV>();
    if (G <= 32) return ex;

    // cross-warp: warp totals through shared memory (one row group per CTA when G > 32)
    const int nw = G >> 5;
    const int w = t >> 5;
    scratch += (threadIdx.x / G) * nw * (NV + 1);  // this row group's slots
    if (pos == 31) {
        scratch[w * (NV + 1)] = v.P;
#pragma unroll
        for (int c = 0; c < NV; ++c) scratch[w * (NV + 1) + 1 + c] = v.B[c];
    }
    __syncthreads();
    Aff<NV> pre = aff_identity<NV>();
    if (!REV) {
        for (int k = 0; k < w; ++k) {
            Aff<NV> e;
            e.P = scratch[k * (NV + 1)];
#pragma unroll
            for (int c = 0; c < NV; ++c) e.B[c] = scratch[k * (NV + 1) + 1 + c];
            pre = aff_compose(pre, e);
        }
    } else {
        for (int k = nw - 1; k > w; --k) {
            Aff<NV> e;
            e.P = scratch[k * (NV + 1)];
#pragma unroll
            for (int c = 0; c < NV; ++c) e.B[c] = scratch[k * (NV + 1) + 1 + c];
            pre = aff_compose(pre, e);
        }
    }
    __syncthreads();  // scratch is reused by the next scan
    return aff_compose(pre, ex);
}

// MINB = 2: two CTAs of <= 320 threads per SM (registers capped accordingly; C_t = 3 rows of
// <= 3840 columns, single-buffered)
// SB: single staging buffer, refilled with the next row group as soon as every thread holds its
// chunk in registers; the outputs leave by direct float4 stores (rows too wide for two
// buffers, and the two-CTAs-per-SM variant).  !SB: double buffer (or, for a single buffer,
// refilled after the bulk stores have read it) and TMA bulk stores.
template <int L, int CT, int MODE, bool SB>
__device__ __forceinline__ void row_pass_body(const RowParams& p);

template <int L, int CT, int MODE>
__global__ void __launch_bounds__(512) k_row_pass(const RowParams p) {
    row_pass_body<L, CT, MODE, false>(p);
}

template <int L, int CT, int MODE>
__global__ void __launch_bounds__(512) k_row_pass_sb(const RowParams p) {
    row_pass_body<L, CT, MODE, true>(p);
}

// two CTAs of <= 320 threads per SM (registers capped at 96): C_t = 3 rows of <= 3840 columns
template <int L, int CT, int MODE>
__global__ void __launch_bounds__(320, 2) k_row_pass2(const RowParams p) {
    row_pass_body<L, CT, MODE, true>(p);
}

template <int L, int CT, int MODE, bool SB>
__device__ __forceinline__ void row_pass_body(const RowParams& p) {
    static_assert(L % 4 == 0, "L must be a multiple of 4 (float4 smem reads)");
    constexpr int NX = (MODE == MODE_SUPPORT) ? 0 : CT;  // input planes (ROWUPD: zbar)
    constexpr int NSLOT = 1 + (MODE == MODE_SUPPORT ? 1 : CT);
    constexpr int NV = (MODE == MODE_SUPPORT) ? 1 : CT;

    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[2];

    const int G = p.G, R = p.R;
    const int rs = threadIdx.x / G;
    const int t = threadIdx.x - rs * G;
    const int64_t bufFloats = (int64_t)R * NSLOT * p.rowstride;
    float* scratch = smem + p.nbuf * bufFloats;  // cross-warp scan scratch (32 * (NV+1) floats)
    const uint32_t rowBytes = (uint32_t)(p.rowlen * sizeof(float));
    const int ngroups = (p.H + R - 1) / R;

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (p.pdl_early) pdl_trigger();
    pdl_wait();  // the previous kernel's output (the row input, Z / T / chat) is complete
    __syncthreads();

    auto issue = [&](int grp, int b) {
        float* buf = smem + b * bufFloats;
        uint32_t bytes = 0;
        for (int q = 0; q < R; ++q)
            if (grp * R + q < p.H) bytes += rowBytes * (1 + NX);
        mbar_arrive_expect_tx(&bar[b], bytes);
        for (int q = 0; q < R; ++q) {
            const int64_t r = (int64_t)grp * R + q;
            if (r >= p.H) break;
            bulk_g2s(buf + (q * NSLOT) * p.rowstride, p.d + r * p.pitch, rowBytes, &bar[b]);
#pragma unroll
            for (int c = 0; c < NX; ++c)
                bulk_g2s(buf + (q * NSLOT + 1 + c) * p.rowstride, p.in + c * p.plane + r * p.pitch, rowBytes,
                         &bar[b]);
            if constexpr (MODE == MODE_ROWUPD) {  // Z, T, chat of that row group into L2
                const uint32_t pb = (uint32_t)(p.W * sizeof(float) + 15) / 16 * 16;
                bulk_prefetch_l2(p.chat + r * p.pitch, pb);
#pragma unroll
                for (int c = 0; c < CT; ++c) {
                    bulk_prefetch_l2(p.Z + c * p.plane + r * p.pitch, pb);
                    bulk_prefetch_l2(p.T + c * p.plane + r * p.pitch, pb);
                }
            }
        }
    };

    int grp = blockIdx.x;
    if (grp < ngroups && threadIdx.x == 0) issue(grp, 0);

    const bool dbl = !SB && p.nbuf == 2;
    for (int it = 0; grp < ngroups; grp += gridDim.x, ++it) {
        const int b = dbl ? (it & 1) : 0;
        const int nxt = grp + gridDim.x;
        if (dbl && threadIdx.x == 0 && nxt < ngroups) {
            bulk_wait_read0();  // stores issued from buffer b^1 have read their smem
            issue(nxt, b ^ 1);
        }
        const int k0 = t * L;
        const int64_t grow = (int64_t)grp * R + rs;  // this thread group's image row
        // ROWUPD: state, target and chat of this row straight from global, coalesced (float4
        // q = j G + t of the row), in flight while the TMA row lands
        constexpr int NQ = (MODE == MODE_ROWUPD) ? L / 4 : 1;
        constexpr int CU = (MODE == MODE_ROWUPD) ? CT : 1;
        float4 zo[CU][NQ], tv[CU][NQ], ch[NQ];
        if constexpr (MODE == MODE_ROWUPD) {
            const bool rok = grow < p.H;
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                const int k = 4 * (j * G + t);
                const bool ok = rok && k < p.W;
                const int64_t o = grow * p.pitch + k;
                const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
                ch[j] = ok ? __ldg(reinterpret_cast<const float4*>(p.chat + o)) : zero;
#pragma unroll
                for (int c = 0; c < CT; ++c) {
                    zo[c][j] = ok ? *reinterpret_cast<const float4*>(p.Z + c * p.plane + o) : zero;
                    tv[c][j] = ok ? __ldg(reinterpret_cast<const float4*>(p.T + c * p.plane + o)) : zero;
                }
            }
        }
        mbar_wait(&bar[b], (uint32_t)(dbl ? ((it >> 1) & 1) : (it & 1)));

        float* row = smem + b * bufFloats + (int64_t)rs * NSLOT * p.rowstride;

        if constexpr (MODE == MODE_ROWUPD) {  // Eq. (3): z <- z - step [lam (z - zbar) + chat (z - t)]
#pragma unroll
            for (int c = 0; c < CT; ++c) {
#pragma unroll
                for (int j = 0; j < NQ; ++j) {
                    const int k = 4 * (j * G + t);
                    if (k < p.W) {
                        float* xs = row + (1 + c) * p.rowstride + k;  // zbar in, new z out (in place)
                        const float4 zb = *reinterpret_cast<const float4*>(xs);
                        const float zz[4] = {zo[c][j].x, zo[c][j].y, zo[c][j].z, zo[c][j].w};
                        const float bb[4] = {zb.x, zb.y, zb.z, zb.w};
                        const float tt[4] = {tv[c][j].x, tv[c][j].y, tv[c][j].z, tv[c][j].w};
                        const float cc[4] = {ch[j].x, ch[j].y, ch[j].z, ch[j].w};
                        float nz[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            nz[u] = fmaf(-p.step, fmaf(p.lam, zz[u] - bb[u], cc[u] * (zz[u] - tt[u])), zz[u]);
                        *reinterpret_cast<float4*>(xs) = make_float4(nz[0], nz[1], nz[2], nz[3]);
                        if (grow < p.H) {
                            float* o = p.Z + c * p.plane + grow * p.pitch + k;
                            if (k + 3 < p.W) {
                                *reinterpret_cast<float4*>(o) = make_float4(nz[0], nz[1], nz[2], nz[3]);
                            } else {
#pragma unroll
                                for (int u = 0; u < 4; ++u)
                                    if (k + u < p.W) o[u] = nz[u];
                            }
                        }
                    }
                }
            }
            __syncthreads();  // the row's new z complete in shared memory
        }

        // ---- load chunk: coefficients A and samples x (masked beyond W) ----
        float A[L];
        float x[NV][L];
#pragma unroll
        for (int j4 = 0; j4 < L; j4 += 4) {
            float4 dv = *reinterpret_cast<const float4*>(row + k0 + j4);
            float dd[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + j4 + u;
                A[j4 + u] = (k < p.W) ? coef_from_d(dd[u], p.kc) : 0.f;
            }
            if constexpr (MODE != MODE_SUPPORT) {
#pragma unroll
                for (int c = 0; c < CT; ++c) {
                    float4 xv = *reinterpret_cast<const float4*>(row + (1 + c) * p.rowstride + k0 + j4);
                    float xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) x[c][j4 + u] = (k0 + j4 + u < p.W) ? xx[u] : 0.f;
                }
            }
        }
        // coefficient linking this chunk's last sample to the next chunk's first
        const int kn = k0 + L;
        const float Anext = (kn < p.W) ? coef_from_d(row[kn], p.kc) : 0.f;
        // single buffer (rows too wide for two): every thread now holds its chunk in registers,
        // so the buffer takes the next row group at once and this group's outputs leave by
        // direct stores (C4 at C_t = 2, 120 KB per row: 445 -> 398 us)
        if constexpr (SB) {
            __syncthreads();
            if (threadIdx.x == 0 && nxt < ngroups) issue(nxt, 0);
        }

        // ---- causal: fold, scan, apply ----
        Aff<NV> m = aff_identity<NV>();
#pragma unroll
        for (int j = 0; j < L; ++j) {
            m.P *= A[j];
#pragma unroll
            for (int c = 0; c < NV; ++c) {
                if constexpr (MODE == MODE_SUPPORT) m.B[c] = fmaf(A[j], m.B[c], 1.f);
                else m.B[c] = fmaf(A[j], m.B[c] - x[c][j], x[c][j]);
            }
        }
        Aff<NV> ex = group_exclusive_scan<NV, false>(m, t, G, scratch);
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            float y = ex.B[c];
#pragma unroll
            for (int j = 0; j < L; ++j) {
                if constexpr (MODE == MODE_SUPPORT) y = fmaf(A[j], y, 1.f);
                else y = fmaf(A[j], y - x[c][j], x[c][j]);
                x[c][j] = y;  // x now holds y (SUPPORT: holds P)
            }
        }

        // ---- anticausal: fold (right to left), reverse scan, apply ----
        m = aff_identity<NV>();
#pragma unroll
        for (int j = L - 1; j >= 0; --j) {
            const float a = (j == L - 1) ? Anext : A[j + 1];
            m.P *= a;
#pragma unroll
            for (int c = 0; c < NV; ++c) {
                if constexpr (MODE == MODE_SUPPORT) m.B[c] = fmaf(a, m.B[c], 1.f);
                else m.B[c] = fmaf(a, m.B[c] - x[c][j], x[c][j]);
            }
        }
        ex = group_exclusive_scan<NV, true>(m, t, G, scratch);

        float* orow = row + p.rowstride;  // output slot(s)
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            float z = ex.B[c];
            float o[L];
#pragma unroll
            for (int j = L - 1; j >= 0; --j) {
                const float a = (j == L - 1) ? Anext : A[j + 1];
                if constexpr (MODE == MODE_SUPPORT) {
                    z = fmaf(a, z, 1.f);
                    o[j] = x[c][j] + z - 1.f;  // s = P + Q - 1
                } else {
                    z = fmaf(a, z - x[c][j], x[c][j]);
                    o[j] = z;
                }
            }
#pragma unroll
            for (int j4 = 0; j4 < L; j4 += 4) {
                const float4 v4 = make_float4(o[j4], o[j4 + 1], o[j4 + 2], o[j4 + 3]);
                if constexpr (SB) {
                    if (grow < p.H && k0 + j4 < p.rowlen)
                        *reinterpret_cast<float4*>(p.out + c * p.plane + grow * p.pitch + k0 + j4) = v4;
                } else {
                    *reinterpret_cast<float4*>(orow + c * p.rowstride + k0 + j4) = v4;
                }
            }
        }

        if constexpr (!SB) {  // the outputs leave through bulk stores from the buffer
            fence_proxy_async_smem();
            __syncthreads();
            if (threadIdx.x == 0) {
                float* buf = smem + b * bufFloats;
                for (int q = 0; q < R; ++q) {
                    const int64_t r = (int64_t)grp * R + q;
                    if (r >= p.H) break;
#pragma unroll
                    for (int c = 0; c < NV; ++c)
                        bulk_s2g(p.out + c * p.plane + r * p.pitch, buf + (q * NSLOT + 1 + c) * p.rowstride,
                                 rowBytes);
                }
                bulk_commit();
                if (!dbl && nxt < ngroups) {  // single buffer: refill once the stores have read it
                    bulk_wait_read0();
                    issue(nxt, 0);
                }
            }
        }
    }
    // the next kernel may launch once every CTA is past its last row group (triggering at the
    // start lets its CTAs take SM resources while this persistent grid runs)
    if (!p.pdl_early) pdl_trigger();
    if (threadIdx.x == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------------------

static const int kLs[] = {4, 12, 20, 36};

cudaError_t plan_row_pass(const Geometry& g, int Ct, int mode, int num_sms, RowPlan* plan, int64_t rowlen) {
    const int nslot = 1 + (mode == MODE_SUPPORT ? 1 : Ct);
    // Narrow rows: the smallest segment length that fits >= 2 rows per CTA (G <= 128).  A
    // row's scan is latency-bound; several rows per CTA keep more of them in flight (C1/C2:
    // row pass 12.7 -> 10.5 us with L = 12 instead of 4); not with L > 12
    // (C3, W = 3840: L = 36 gave 84.7 us against 51.6 at L = 12).  Wide rows: the smallest L >= 12
    // with G <= 512 (one row per CTA, the segment loads coalesce either way).
    int L = 0, G = 0;
    const int forced = option_row_seg();  // experiments: a forced segment length
    if (forced > 0 && (g.W + forced - 1) / forced <= 512) {
        L = forced;
        G = (int)((g.W + forced - 1) / forced);
    }
    for (int lim : {128, 512}) {
        if (G) break;
        for (int cand : kLs) {
            if (lim == 128 && cand > 12) break;  // long segments cost more than they save
            // wide rows never take 4 samples per thread (512 threads per row at W = 2000: row pass
            // 88 us against 54 at 12 samples, C_t = 1, H = 10000; 1920 x 1080 x 3: 25 -> 19 us)
            if (lim == 512 && cand < 12) continue;
            int64_t need = (g.W + cand - 1) / cand;
            if (need <= lim) {
                L = cand;
                G = (int)need;
                break;
            }
        }
        if (G) break;
    }
    if (G == 0) return cudaErrorInvalidValue;  // W > 36 * 512
    if (G <= 32) {
        int p2 = 1;
        while (p2 < G) p2 <<= 1;
        G = p2;
    } else {
        G = (G + 31) / 32 * 32;
    }
    int R = G >= 256 ? 1 : 256 / G;
    if (R > g.H) R = (int)g.H;
    if (R < 1) R = 1;
    plan->L = L;
    plan->G = G;
    plan->R = R;
    plan->threads = G * R;
    const int64_t rl = rowlen > 0 ? rowlen : g.pitch;
    int64_t rs = rl > (int64_t)G * L ? rl : (int64_t)G * L;
    rs = (rs + 3) / 4 * 4;
    plan->rowstride = rs;
    plan->rowlen = rl;
    plan->nbuf = 2;
    plan->smem = (size_t)2 * R * nslot * rs * sizeof(float) + 32 * 8 * sizeof(float);
    if (plan->smem > 227 * 1024) {  // very wide rows: one buffer (no prefetch overlap)
        plan->nbuf = 1;
        plan->smem = (size_t)R * nslot * rs * sizeof(float) + 32 * 8 * sizeof(float);
    }
    if (plan->smem > 227 * 1024) return cudaErrorInvalidValue;
    plan->minb = 1;
    if (Ct == 3 && L == 12 && mode == MODE_FILTER && plan->threads <= 320 && row_minb2()) {
        // C_t = 3 rows of <= 3840 columns: two single-buffered CTAs per SM instead of one
        // double-buffered one (registers capped at 96 per thread).  Batched C3 row pass 0.353
        // -> 0.335 ms; not the fused row update (0.688 -> 0.827 ms), which plans as ROWUPD
        plan->minb = 2;
        plan->nbuf = 1;
        plan->smem = (size_t)R * nslot * rs * sizeof(float) + 32 * 8 * sizeof(float);
    }
    const int64_t ngroups = (g.H + R - 1) / R;
    int per_sm = 1;
    // occupancy limited by threads and smem
    int by_threads = 2048 / plan->threads;
    int by_smem = (int)((228 * 1024) / (plan->smem + 1024));
    per_sm = by_threads < by_smem ? by_threads : by_smem;
    if (plan->minb == 2 && per_sm > 2) per_sm = 2;  // what the register cap allows
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)num_sms * per_sm;
    if (grid > ngroups) grid = ngroups;
    plan->grid = (int)grid;
    return cudaSuccess;
}

// PDL trigger at the end of the kernel (option pdl = 2: at the start, for experiments)
static int row_pdl_early(const RowPlan& plan, const Geometry& g) {
    (void)plan;
    (void)g;
    return option_pdl() == 2;
}

template <int L, int CT, int MODE>
static cudaError_t launch_t(const RowPlan& plan, const RowParams& p, cudaStream_t s) {
    if constexpr (L == 12 && CT == 3 && MODE != MODE_SUPPORT) {
        if (plan.minb == 2) {
            cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k_row_pass2<L, CT, MODE>), plan.smem);
            if (e != cudaSuccess) return e;
            return launch_pdl(k_row_pass2<L, CT, MODE>, dim3(plan.grid), dim3(plan.threads), plan.smem, s, p);
        }
    }
    if (plan.nbuf == 1) {  // one buffer: the early-refill variant
        cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k_row_pass_sb<L, CT, MODE>), plan.smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(k_row_pass_sb<L, CT, MODE>, dim3(plan.grid), dim3(plan.threads), plan.smem, s, p);
    }
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k_row_pass<L, CT, MODE>), plan.smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(k_row_pass<L, CT, MODE>, dim3(plan.grid), dim3(plan.threads), plan.smem, s, p);
}

template <int L, int MODE>
static cudaError_t launch_ct(const RowPlan& plan, const RowParams& p, int Ct, cudaStream_t s) {
    switch (Ct) {
        case 1: return launch_t<L, 1, MODE>(plan, p, s);
        case 2: return launch_t<L, 2, MODE>(plan, p, s);
        case 3: return launch_t<L, 3, MODE>(plan, p, s);
        case 4: return launch_t<L, 4, MODE>(plan, p, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_row_update(const RowPlan& plan, const Geometry& g, int Ct, const float* zbar, float* out,
                              const float* d, float kc, const UpdateArgs& u, cudaStream_t s) {
    RowParams p = {};
    p.in = zbar;
    p.out = out;
    p.d = d;
    p.Z = u.Z;
    p.T = u.T;
    p.chat = u.chat;
    p.lam = u.lam;
    p.step = u.step;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.rowstride = plan.rowstride;
    p.rowlen = plan.rowlen;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.G = plan.G;
    p.R = plan.R;
    p.nbuf = plan.nbuf;
    p.kc = kc;
    p.pdl_early = row_pdl_early(plan, g);
    switch (plan.L) {
        case 4: return launch_ct<4, MODE_ROWUPD>(plan, p, Ct, s);
        case 12: return launch_ct<12, MODE_ROWUPD>(plan, p, Ct, s);
        case 20: return launch_ct<20, MODE_ROWUPD>(plan, p, Ct, s);
        case 36: return launch_ct<36, MODE_ROWUPD>(plan, p, Ct, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_row_pass(const RowPlan& plan, const Geometry& g, int Ct, int mode, const float* in, float* out,
                            const float* d, float kc, cudaStream_t s) {
    RowParams p = {};
    p.in = in;
    p.out = out;
    p.d = d;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.rowstride = plan.rowstride;
    p.rowlen = plan.rowlen;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.G = plan.G;
    p.R = plan.R;
    p.nbuf = plan.nbuf;
    p.kc = kc;
    p.pdl_early = row_pdl_early(plan, g);
    if (mode == MODE_SUPPORT) {
        switch (plan.L) {
            case 4: return launch_t<4, 1, MODE_SUPPORT>(plan, p, s);
            case 12: return launch_t<12, 1, MODE_SUPPORT>(plan, p, s);
            case 20: return launch_t<20, 1, MODE_SUPPORT>(plan, p, s);
            case 36: return launch_t<36, 1, MODE_SUPPORT>(plan, p, s);
        }
        return cudaErrorInvalidValue;
    }
    switch (plan.L) {
        case 4: return launch_ct<4, MODE_FILTER>(plan, p, Ct, s);
        case 12: return launch_ct<12, MODE_FILTER>(plan, p, Ct, s);
        case 20: return launch_ct<20, MODE_FILTER>(plan, p, Ct, s);
        case 36: return launch_ct<36, MODE_FILTER>(plan, p, Ct, s);
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------
// Row strips (images wider than one CTA's staging buffer holds).  The
// row pass runs on vertical strips [c_b, c_{b+1}) with a zero carry at each strip's left edge
// and the link to its right cut; the seams are fixed up afterwards with per-row edge profiles:
// the row-strip algebra of the column passes (reading R26) along x.  Seam j (1 <= j < n) lies
// between strips j - 1 and j at column c_j; profiles are [seam][row][L].

// how many columns a carry entering a strip keeps an influence >= 2^-26 of itself (max over
// rows, from the left edge of strip j and from the right edge of strip j - 1)
__global__ void k_row_edge_length(const float* __restrict__ d, int64_t H, int64_t pitch, RowStrips st, int Lcap,
                                  float kc, unsigned* __restrict__ len) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y + 1;
    if (r >= H) return;
    const float thr = 1.0f / 67108864.0f;  // 2^-26
    const float* dr = d + r * pitch + st.c[j];
    float G = 1.f;
    int k = 0;
    for (; k < Lcap; ++k) {
        G *= coef_from_d(__ldg(dr + k), kc);
        if (G < thr) break;
    }
    atomicMax(&len[0], (unsigned)k);
    float Th = 1.f;
    int m = 0;
    for (; m < Lcap; ++m) {
        Th *= coef_from_d(__ldg(dr - m), kc);
        if (Th < thr) break;
    }
    atomicMax(&len[1], (unsigned)m);
}

// Gamma (the first L columns of strip j: G_k = prod_{m <= k} a_{c_j + m}, then its anticausal
// response unless raw) and Theta (the last L columns of strip j - 1: the product of the links
// from column k + 1 to c_j), thread per (row, seam)
__global__ void k_row_edge_profiles(const float* __restrict__ d, int64_t H, int64_t pitch, RowStrips st, int L,
                                    float kc, float* __restrict__ gam, float* __restrict__ theta, bool raw) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y + 1;
    if (r >= H) return;
    const float* dr = d + r * pitch + st.c[j];
    float* gm = gam + ((int64_t)(j - 1) * H + r) * L;
    float* th = theta + ((int64_t)(j - 1) * H + r) * L;
    float G = 1.f;
    for (int k = 0; k < L; ++k) {
        G *= coef_from_d(__ldg(dr + k), kc);
        gm[k] = G;
    }
    float dz = 0.f;
    for (int k = L - 1; k >= 0 && !raw; --k) {
        const float an = coef_from_d(__ldg(dr + k + 1), kc);
        dz = fmaf(an, dz - gm[k], gm[k]);
        gm[k] = dz;
    }
    float t = coef_from_d(__ldg(dr), kc);  // the link across the seam
    for (int k = L - 1; k >= 0; --k) {     // theta[k]: column c_j - L + k
        th[k] = t;
        t *= coef_from_d(__ldg(dr - (L - k)), kc);
    }
}

// block per (row, seam): every plane's y_last = x[c_j - 1] and z0 = x[c_j] are read before any
// thread writes; then x[c_j + k] += y_last Gamma[k] and x[c_j - L + k] += e Theta[k], with
// e = z0 + y_last Gamma[0] - y_last (raw, the support: c = s0[c_j - 1], e = s0[c_j])
// x points at row r0 of plane 0; the profiles hold Hp rows
__global__ void __launch_bounds__(128) k_row_seam_fix(float* __restrict__ x, int Ct, int64_t pitch, int64_t plane,
                                                      RowStrips st, int L, const float* __restrict__ gam,
                                                      const float* __restrict__ theta, int64_t Hp, int64_t r0,
                                                      bool raw) {
    const int64_t r = blockIdx.x;
    const int j = blockIdx.y + 1;
    pdl_wait();
    const int64_t cj = st.c[j];
    const float* gm = gam + ((int64_t)(j - 1) * Hp + r0 + r) * L;
    const float* th = theta + ((int64_t)(j - 1) * Hp + r0 + r) * L;
    float yl[4], e[4];
    const float g0 = __ldg(gm);
    for (int v = 0; v < Ct && v < 4; ++v) {
        const float* xr = x + v * plane + r * pitch;
        yl[v] = xr[cj - 1];
        const float z0 = xr[cj];
        e[v] = raw ? z0 : fmaf(yl[v], g0, z0) - yl[v];
    }
    __syncthreads();
    for (int v = 0; v < Ct && v < 4; ++v) {
        float* xr = x + v * plane + r * pitch;
        for (int k = threadIdx.x; k < 2 * L; k += blockDim.x) {
            if (k < L) xr[cj + k] = fmaf(yl[v], __ldg(gm + k), xr[cj + k]);
            else xr[cj - 2 * L + k] = fmaf(e[v], __ldg(th + (k - L)), xr[cj - 2 * L + k]);
        }
    }
}

cudaError_t launch_row_edge_length(const float* d, const Geometry& g, const RowStrips& st, int Lcap, float kc,
                                   unsigned* len, cudaStream_t s) {
    if (st.n < 2) return cudaSuccess;
    k_row_edge_length<<<dim3((unsigned)((g.H + 127) / 128), (unsigned)(st.n - 1)), 128, 0, s>>>(d, g.H, g.pitch, st,
                                                                                                 Lcap, kc, len);
    return cudaGetLastError();
}

cudaError_t launch_row_edge_profiles(const float* d, const Geometry& g, const RowStrips& st, int L, float kc,
                                     float* gam, float* theta, bool raw, cudaStream_t s) {
    if (st.n < 2) return cudaSuccess;
    k_row_edge_profiles<<<dim3((unsigned)((g.H + 127) / 128), (unsigned)(st.n - 1)), 128, 0, s>>>(
        d, g.H, g.pitch, st, L, kc, gam, theta, raw);
    return cudaGetLastError();
}

cudaError_t launch_row_seam_fix(float* x, int Ct, const Geometry& g, const RowStrips& st, int L, const float* gam,
                                const float* theta, int64_t Hp, int64_t r0, bool raw, cudaStream_t s) {
    if (st.n < 2 || g.H < 1) return cudaSuccess;
    if (Ct > 4) return cudaErrorInvalidValue;
    return launch_pdl(k_row_seam_fix, dim3((unsigned)g.H, (unsigned)(st.n - 1)), dim3(128), 0, s, x, Ct, g.pitch,
                      g.plane, st, L, gam, theta, Hp, r0, raw);
}

}  // namespace dts
