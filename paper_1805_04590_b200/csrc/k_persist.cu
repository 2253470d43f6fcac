// k_persist.cu -- the whole DTS solve of an L2-RESIDENT image in ONE persistent kernel
// (sm_100a).  For the paper's own workload shapes (stereo refinement 1400 x 1000, P:473-481;
// 16x depth SR 1376 x 1024) the working set (X, Z, T, chat, d_x, A1 ~ 34 MB)
// lives in the 126 MB L2, and a pass over it is a few microseconds of L2 traffic: launching
// one kernel per pass (7 launches per iteration) made those solves launch- and ramp-bound.
//
// Same arithmetic as the streaming kernels (readings R4-R12):
//   for k = 0 .. iters-1, i = 1..N:
//     row phase i:     X <- RF_rows(i == 1 ? Z : X, a_i^{d_x})   (i == 1, k > 0: the Eq. (3) step
//                      of iteration k-1 is applied to Z first, elementwise, as in k_row.cu ROWUPD)
//     column phase i:  X <- RF_cols(X, a_i^{d_y})                (a_i^{d_y} = A1^(2^(i-1)), R5)
//   epilogue:          out <- Z - step [lambda (Z - X) + chat (Z - T)]
// Work decomposition (fixed for the whole launch; every warp is resident -- cooperative launch):
//   row phase:    one warp per image row, staged through shared memory with coalesced loads;
//                 lane l holds the L consecutive samples [l L, l L + L) in registers; causal
//                 fold -> warp shuffle scan -> exact apply, anticausal the same way (the
//                 k_row.cu scheme with a 32-thread row group).
//   column phase: one CTA per (32-column tile, band of 16 segments of LS rows); lane =
//                 column, warp = segment, LS rows in registers.  The segment maps of a band are
//                 scanned in shared memory; band totals are published to L2 with a per-phase
//                 epoch flag, and a band composes the totals of the bands above it (causal
//                 carry) and, after its anticausal fold, those below it (anticausal carry).
//                 Every total is published before its CTA waits on anything: no wait cycle.
//   between phases: a software grid barrier (all CTAs are co-resident by construction).
// Every wait spins with a bound and traps instead of hanging the GPU.
#include "dts_device.cuh"
#include "dts_launch.h"

#include <mutex>
#include <vector>

namespace dts {
namespace pers {

constexpr int THREADS = 512;  // 16 warps, one CTA per SM (<= 128 registers per thread)
constexpr long long SPIN_LIMIT = 1ll << 27;

struct Params {
    float* X;
    float* Z;
    const float* T;
    const float* chat;
    const float* dx;   // d_x; row coefficients a_i^{d_x} = 2^(-kc_i d_x)
    const float* A1y;  // A1 = a_1^{d_y}, rows 0..H (row H = 0: the image bottom)
    float* out;        // H x W, row-major (C_t = 1)
    unsigned* resid;   // optional [iters]: ||g_k||_inf as float bits (atomicMax; g >= 0 bits order)
    float* maps;       // [ntiles][nseg][4][32]: causal (P, B), anticausal (Q, E)
    unsigned* flags;   // [ntiles][nseg][2]
    unsigned long long* bar;  // monotonic arrival counter of the grid barrier
    unsigned long long bar_base;  // its value when this launch starts
    int64_t pitch;
    int H, W, N, iters, ntiles, nseg;
    unsigned epoch0;
    float kc[4];
    float lam, step;
    unsigned long long* timers;  // debug (nullable): block 0 stamps %globaltimer at every phase boundary
};

__device__ __forceinline__ void substamp(const Params& p, int slot) {
    if (p.timers && blockIdx.x == 0 && threadIdx.x == 0 && p.timers[3000 + slot] == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.timers[3000 + slot] = t;
    }
}

__device__ __forceinline__ void stamp(const Params& p, int& n) {
    if (p.timers && blockIdx.x == 0 && threadIdx.x == 0 && n < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.timers[n] = t;
    }
    ++n;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// software grid barrier on a monotonic 64-bit arrival counter: barrier number b of a launch
// completes when the counter reaches base + (b + 1) * gridDim.x (base: the counter value at
// launch, tracked by the host; launches on a context are stream-ordered).  The arrival is a
// release (it publishes the CTA's writes, ordered before it by __syncthreads), the poll an
// acquire.  Cross-CTA data is read with ld.global.cg (L2) and read-only data never changes
// inside a launch, so no L1 invalidation is needed.
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        long long it = 0;
        while (ld_acquire64(bar) < target) {
            if (++it > SPIN_LIMIT) __trap();
            if (it > 256) __nanosleep(16);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned want) {
    long long it = 0;
    while (ld_acquire(f) != want) {
        if (++it > SPIN_LIMIT) __trap();
        if (it > 256) __nanosleep(16);
    }
}

// Eq. (3), the k_update arithmetic
__device__ __forceinline__ float eq3(float z, float zb, float t, float ch, float lam, float step, float& gabs) {
    const float g = fmaf(lam, z - zb, ch * (z - t));
    gabs = fmaxf(gabs, fabsf(g));
    return fmaf(-step, g, z);
}

__device__ __forceinline__ void resid_max(unsigned* resid, int k, float gabs) {
    if (!resid) return;
    const unsigned m = __reduce_max_sync(FULL, __float_as_uint(gabs));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(resid + k, m);
}

// exclusive scan of affine maps over the 32 lanes (REV: from lane 31 downwards)
template <bool REV>
__device__ __forceinline__ void warp_exscan(float& P, float& B) {
    const int lane = threadIdx.x & 31;
    const int pos = REV ? 31 - lane : lane;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float eP = REV ? __shfl_down_sync(FULL, P, off) : __shfl_up_sync(FULL, P, off);
        const float eB = REV ? __shfl_down_sync(FULL, B, off) : __shfl_up_sync(FULL, B, off);
        if (pos >= off) {  // earlier map e, then this one
            B = fmaf(P, eB, B);
            P = eP * P;
        }
    }
    float xP = REV ? __shfl_down_sync(FULL, P, 1) : __shfl_up_sync(FULL, P, 1);
    float xB = REV ? __shfl_down_sync(FULL, B, 1) : __shfl_up_sync(FULL, B, 1);
    if (pos == 0) {
        xP = 1.f;
        xB = 0.f;
    }
    P = xP;
    B = xB;
}

// ---- row phase: warp per row, L samples per lane ---------------------------------------
// A row arrives in the warp's shared-memory slot with coalesced float4 loads (lane-
// contiguous), laid out chunk by chunk with 4 floats of skew per L-sample chunk so that the
// per-lane float4 reads of a chunk are bank-conflict free; results leave the same way.
template <int L>
__device__ __forceinline__ void row_phase(const Params& p, int pass, int k, int gwarp, int nwarps, float* wsm) {
    static_assert(L % 4 == 0, "float4 chunks");
    constexpr int LP = L + 4;
    float* sx = wsm;
    float* sd = wsm + 32 * LP;
    const int lane = threadIdx.x & 31;
    const float kc = p.kc[pass];
    const bool fromZ = pass == 0;
    const bool upd = fromZ && k > 0;
    const int nq = (p.W + 3) >> 2;  // float4 per row (the pitch is a multiple of 32)
    const int k0 = lane * L;
    float gabs = 0.f;
    for (int r = gwarp; r < p.H; r += nwarps) {
        const int64_t ro = (int64_t)r * p.pitch;
        for (int q = lane; q < nq; q += 32) {
            const int e = q << 2;
            const int si = e + (e / L) * 4;
            const float4 dv = ldg4(p.dx + ro + e);
            float4 xv;
            if (fromZ) {
                xv = ldcg4(p.Z + ro + e);
                if (upd) {  // Eq. (3) of iteration k-1 (zbar = X), written back to Z
                    const float4 zb = ldcg4(p.X + ro + e);
                    const float4 tv = ldg4(p.T + ro + e);
                    const float4 ch = ldg4(p.chat + ro + e);
                    float gx = 0.f, gy = 0.f, gz = 0.f, gw = 0.f;
                    xv.x = eq3(xv.x, zb.x, tv.x, ch.x, p.lam, p.step, gx);
                    xv.y = eq3(xv.y, zb.y, tv.y, ch.y, p.lam, p.step, gy);
                    xv.z = eq3(xv.z, zb.z, tv.z, ch.z, p.lam, p.step, gz);
                    xv.w = eq3(xv.w, zb.w, tv.w, ch.w, p.lam, p.step, gw);
                    gabs = fmaxf(gabs, gx);
                    if (e + 1 < p.W) gabs = fmaxf(gabs, gy);
                    if (e + 2 < p.W) gabs = fmaxf(gabs, gz);
                    if (e + 3 < p.W) gabs = fmaxf(gabs, gw);
                    *reinterpret_cast<float4*>(p.Z + ro + e) = xv;
                }
            } else {
                xv = ldcg4(p.X + ro + e);
            }
            *reinterpret_cast<float4*>(sd + si) = dv;
            *reinterpret_cast<float4*>(sx + si) = xv;
        }
        __syncwarp();
        float A[L], x[L];
#pragma unroll
        for (int j4 = 0; j4 < L; j4 += 4) {
            const float4 dv = *reinterpret_cast<const float4*>(sd + lane * LP + j4);
            const float4 xv = *reinterpret_cast<const float4*>(sx + lane * LP + j4);
            const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
            const float xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool ok = k0 + j4 + u < p.W;  // masks the tail and the unwritten chunks
                A[j4 + u] = ok ? coef_from_d(dd[u], kc) : 0.f;
                x[j4 + u] = ok ? xx[u] : 0.f;
            }
        }
        // coefficient linking this chunk's last sample to the next lane's first (0 past W)
        float Anext = __shfl_down_sync(FULL, A[0], 1);
        if (lane == 31) Anext = 0.f;

        // causal: fold, scan, apply
        float P = 1.f, B = 0.f;
#pragma unroll
        for (int j = 0; j < L; ++j) {
            P *= A[j];
            B = fmaf(A[j], B - x[j], x[j]);
        }
        warp_exscan<false>(P, B);
        float y = B;
#pragma unroll
        for (int j = 0; j < L; ++j) {
            y = fmaf(A[j], y - x[j], x[j]);
            x[j] = y;
        }
        // anticausal: the step at j uses A[j + 1]
        P = 1.f;
        B = 0.f;
#pragma unroll
        for (int j = L - 1; j >= 0; --j) {
            const float a = (j == L - 1) ? Anext : A[j + 1];
            P *= a;
            B = fmaf(a, B - x[j], x[j]);
        }
        warp_exscan<true>(P, B);
        float z = B;
#pragma unroll
        for (int j = L - 1; j >= 0; --j) {
            const float a = (j == L - 1) ? Anext : A[j + 1];
            z = fmaf(a, z - x[j], x[j]);
            x[j] = z;
        }
#pragma unroll
        for (int j4 = 0; j4 < L; j4 += 4)
            *reinterpret_cast<float4*>(sx + lane * LP + j4) = make_float4(x[j4], x[j4 + 1], x[j4 + 2], x[j4 + 3]);
        __syncwarp();
        for (int q = lane; q < nq; q += 32) {
            const int e = q << 2;
            *reinterpret_cast<float4*>(p.X + ro + e) = *reinterpret_cast<const float4*>(sx + e + (e / L) * 4);
        }
        __syncwarp();  // the slot is reused by the next row
    }
    if (upd) resid_max(p.resid, k - 1, gabs);
}

// ---- column phase: CTA per (32-column tile, band of 16 LS-row segments) ---------------
// lane = column, warp s = segment s of the band, LS rows in registers.  Inside the CTA the
// 16 segment maps of each column are scanned with half-warp shuffles (two columns per
// warp); the band's total map is published to L2 with a per-phase epoch flag, and warp 0
// composes the totals of the bands above (causal carry) or below (anticausal carry).
// Every total is published before its CTA waits on anything, so no wait cycle exists.
constexpr int SEGS = THREADS / 32;  // segments per band

// exclusive scan of the SEGS maps (P at seg[0][s], B at seg[1][s], stride 33) of columns cA (lanes
// 0-15) and cB (lanes 16-31); REV: from the last segment upwards; the band total -> tot[2][32]
template <bool REV>
__device__ __forceinline__ void band_scan(float* seg, int cA, int cB, float* tot) {
    const int lane = threadIdx.x & 31;
    const int sl = lane & 15;
    const int cc = lane < 16 ? cA : cB;
    float P = seg[sl * 33 + cc];
    float B = seg[SEGS * 33 + sl * 33 + cc];
    const int pos = REV ? 15 - sl : sl;
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        const float eP = REV ? __shfl_down_sync(FULL, P, off, 16) : __shfl_up_sync(FULL, P, off, 16);
        const float eB = REV ? __shfl_down_sync(FULL, B, off, 16) : __shfl_up_sync(FULL, B, off, 16);
        if (pos >= off) {
            B = fmaf(P, eB, B);
            P = eP * P;
        }
    }
    float xP = REV ? __shfl_down_sync(FULL, P, 1, 16) : __shfl_up_sync(FULL, P, 1, 16);
    float xB = REV ? __shfl_down_sync(FULL, B, 1, 16) : __shfl_up_sync(FULL, B, 1, 16);
    if (pos == 0) {
        xP = 1.f;
        xB = 0.f;
    }
    seg[sl * 33 + cc] = xP;
    seg[SEGS * 33 + sl * 33 + cc] = xB;
    if (pos == 15) {
        tot[cc] = P;
        tot[32 + cc] = B;
    }
}

template <int LS>
__device__ __forceinline__ void col_phase(const Params& p, int pass, unsigned epC, unsigned epA, float* sm) {
    const int nbands = p.nseg;  // bands per tile
    const int task = blockIdx.x;
    if (task >= p.ntiles * nbands) return;  // CTA-uniform
    float* seg = sm;                  // [2][SEGS][33]
    float* tot = sm + 2 * SEGS * 33;  // [2][32]
    float* carry = tot + 64;          // [32]
    const int lane = threadIdx.x & 31;
    const int s = threadIdx.x >> 5;
    const int tile = task / nbands;
    const int band = task - tile * nbands;
    const int col = tile * 32 + lane;  // < pitch: lanes past W work on the row padding, never stored
    const int r0 = (band * SEGS + s) * LS;
    const int nsq = pass;  // a_i = A1^(2^(i-1)) (R5: sigma halves per pass)
    auto coef = [&](float a1) {
        for (int q = 0; q < nsq; ++q) a1 *= a1;
        return a1;
    };
    float a[LS], x[LS];
    const float* ap = p.A1y + (int64_t)r0 * p.pitch + col;
    float* xp = p.X + (int64_t)r0 * p.pitch + col;
    if (r0 + LS <= p.H) {
#pragma unroll
        for (int j = 0; j < LS; ++j) {
            a[j] = coef(__ldg(ap + (int64_t)j * p.pitch));
            x[j] = __ldcg(xp + (int64_t)j * p.pitch);
        }
    } else {
#pragma unroll
        for (int j = 0; j < LS; ++j) {
            const bool ok = r0 + j < p.H;
            a[j] = ok ? coef(__ldg(ap + (int64_t)j * p.pitch)) : 0.f;
            x[j] = ok ? __ldcg(xp + (int64_t)j * p.pitch) : 0.f;
        }
    }
    // link of the segment's last row to the next row (A1 row H is 0: the image bottom)
    const float anext = (r0 + LS <= p.H) ? coef(__ldg(ap + (int64_t)LS * p.pitch)) : 0.f;
    float* mp = p.maps + (int64_t)tile * nbands * 128;  // this tile's band totals
    unsigned* fl = p.flags + (int64_t)tile * nbands * 2;

    substamp(p, 0);
    // 1. causal fold -> band scan -> publish the band total
    {
        float P = 1.f, B = 0.f;
#pragma unroll
        for (int j = 0; j < LS; ++j) {
            P *= a[j];
            B = fmaf(a[j], B - x[j], x[j]);
        }
        seg[s * 33 + lane] = P;
        seg[SEGS * 33 + s * 33 + lane] = B;
    }
    __syncthreads();
    substamp(p, 1);
    band_scan<false>(seg, s, s + 16, tot);
    __syncthreads();
    substamp(p, 2);
    if (s == 0) {
        mp[band * 128 + lane] = tot[lane];
        mp[band * 128 + 32 + lane] = tot[32 + lane];
        __syncwarp();
        if (lane == 0) st_release(fl + band * 2 + 0, epC);  // cumulative: the warp's stores precede it
        // causal carry into the band: the totals of the bands above, in order
        for (int q0 = 0; q0 < band; q0 += 32)
            if (q0 + lane < band) wait_flag(fl + (q0 + lane) * 2 + 0, epC);
        __syncwarp();
        float c = 0.f;
        for (int q = 0; q < band; ++q) c = fmaf(__ldcg(mp + q * 128 + lane), c, __ldcg(mp + q * 128 + 32 + lane));
        carry[lane] = c;
    }
    __syncthreads();
    substamp(p, 3);
    // 2. exact causal apply (segment prefix applied to the band carry), anticausal fold
    {
        float y = fmaf(seg[s * 33 + lane], carry[lane], seg[SEGS * 33 + s * 33 + lane]);
#pragma unroll
        for (int j = 0; j < LS; ++j) {
            y = fmaf(a[j], y - x[j], x[j]);
            x[j] = y;
        }
        float Q = 1.f, E = 0.f;
#pragma unroll
        for (int j = LS - 1; j >= 0; --j) {
            const float an = (j == LS - 1) ? anext : a[j + 1];
            Q *= an;
            E = fmaf(an, E - x[j], x[j]);
        }
        __syncthreads();  // every warp has read its causal prefix
        seg[s * 33 + lane] = Q;
        seg[SEGS * 33 + s * 33 + lane] = E;
    }
    __syncthreads();
    band_scan<true>(seg, s, s + 16, tot);
    __syncthreads();
    substamp(p, 4);
    if (s == 0) {
        mp[band * 128 + 64 + lane] = tot[lane];
        mp[band * 128 + 96 + lane] = tot[32 + lane];
        __syncwarp();
        if (lane == 0) st_release(fl + band * 2 + 1, epA);
        // anticausal carry: the totals of the bands below, bottom first
        for (int q0 = band + 1; q0 < nbands; q0 += 32)
            if (q0 + lane < nbands) wait_flag(fl + (q0 + lane) * 2 + 1, epA);
        __syncwarp();
        float e = 0.f;
        for (int q = nbands - 1; q > band; --q)
            e = fmaf(__ldcg(mp + q * 128 + 64 + lane), e, __ldcg(mp + q * 128 + 96 + lane));
        carry[lane] = e;
    }
    __syncthreads();
    substamp(p, 5);
    // 3. exact anticausal apply, store
    {
        float z = fmaf(seg[s * 33 + lane], carry[lane], seg[SEGS * 33 + s * 33 + lane]);
#pragma unroll
        for (int j = LS - 1; j >= 0; --j) {
            const float an = (j == LS - 1) ? anext : a[j + 1];
            z = fmaf(an, z - x[j], x[j]);
            x[j] = z;
        }
    }
    if (r0 + LS <= p.H) {
#pragma unroll
        for (int j = 0; j < LS; ++j) xp[(int64_t)j * p.pitch] = x[j];
    } else {
#pragma unroll
        for (int j = 0; j < LS; ++j)
            if (r0 + j < p.H) xp[(int64_t)j * p.pitch] = x[j];
    }
    substamp(p, 6);
}

template <int L>
constexpr size_t smem_bytes() {
    const size_t rows = (size_t)(THREADS / 32) * 2 * 32 * (L + 4) * sizeof(float);
    const size_t cols = (size_t)(2 * SEGS * 33 + 96) * sizeof(float);
    return rows > cols ? rows : cols;
}

template <int L, int LS>
__global__ void __launch_bounds__(THREADS, 1) k_solve_persist(const Params p) {
    extern __shared__ __align__(16) float sm[];
    unsigned long long target = p.bar_base;
    const int wpb = THREADS / 32;
    // warp w of CTA b takes rows b + w * gridDim.x, ...: every SM gets a share of the rows
    const int gwarp = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    const int nwarps = gridDim.x * wpb;
    int nst = 0;
    stamp(p, nst);
    for (int k = 0; k < p.iters; ++k) {
        for (int i = 0; i < p.N; ++i) {
            row_phase<L>(p, i, k, gwarp, nwarps, sm + (threadIdx.x >> 5) * 2 * 32 * (L + 4));
            stamp(p, nst);
            grid_sync(p.bar, target);
            stamp(p, nst);
            const unsigned epC = p.epoch0 + 2u * (unsigned)(k * p.N + i);
            col_phase<LS>(p, i, epC, epC + 1u, sm);
            stamp(p, nst);
            grid_sync(p.bar, target);
            stamp(p, nst);
        }
    }
    // epilogue: the last iteration's Eq. (3) step into the row-major output
    float gabs = 0.f;
    const int lane = threadIdx.x & 31;
    for (int r = gwarp; r < p.H; r += nwarps) {
        const int64_t ro = (int64_t)r * p.pitch;
        for (int c = lane; c < p.W; c += 32) {
            const float z = __ldcg(p.Z + ro + c);
            p.out[(int64_t)r * p.W + c] =
                eq3(z, __ldcg(p.X + ro + c), __ldg(p.T + ro + c), __ldg(p.chat + ro + c), p.lam, p.step, gabs);
        }
    }
    resid_max(p.resid, p.iters - 1, gabs);
}

template <int L, int LS>
static const void* kfn() {
    return reinterpret_cast<const void*>(k_solve_persist<L, LS>);
}

static const void* kernel_for(int L, int LS) {
    switch (L * 100 + LS) {
        case 1616: return kfn<16, 16>();
        case 1624: return kfn<16, 24>();
        case 1632: return kfn<16, 32>();
        case 1648: return kfn<16, 48>();
        case 3216: return kfn<32, 16>();
        case 3224: return kfn<32, 24>();
        case 3232: return kfn<32, 32>();
        case 3248: return kfn<32, 48>();
        case 4816: return kfn<48, 16>();
        case 4824: return kfn<48, 24>();
        case 4832: return kfn<48, 32>();
        case 4848: return kfn<48, 48>();
    }
    return nullptr;
}

}  // namespace pers

// debug hook (tools/probe_persist.py via dts_debug_persist_timers): device buffer of 4096 stamps
static unsigned long long* g_timers = nullptr;
unsigned long long* persist_timers() { return g_timers; }
void set_persist_timers(unsigned long long* t) { g_timers = t; }

static size_t smem_for(int L) {
    return L == 16 ? pers::smem_bytes<16>() : (L == 32 ? pers::smem_bytes<32>() : pers::smem_bytes<48>());
}

// Plan: C_t = 1, N <= 4 (columns square A1), W <= 1536 (one warp holds a row), and every
// column-phase task (32-column tile x band of 16 LS-row segments) has its own resident CTA.
cudaError_t plan_persist(const Geometry& g, int Ct, int N, int num_sms, PersistPlan* plan) {
    if (Ct != 1 || N < 1 || N > 4 || g.W > 1536 || g.H < 1) return cudaErrorNotSupported;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int coop = 0;
    if ((e = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev)) != cudaSuccess) return e;
    if (!coop) return cudaErrorNotSupported;
    const int L = g.W <= 512 ? 16 : (g.W <= 1024 ? 32 : 48);
    const size_t smem = smem_for(L);
    const int ntiles = (int)((g.W + 31) / 32);
    for (int LS : {16, 24, 32, 48}) {
        const void* fn = pers::kernel_for(L, LS);
        if ((e = ensure_smem_attr(fn, smem)) != cudaSuccess) return e;
        int per_sm = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, pers::THREADS, smem)) != cudaSuccess)
            return e;
        if (per_sm < 1) continue;
        const int64_t nbands = (g.H + (int64_t)pers::SEGS * LS - 1) / ((int64_t)pers::SEGS * LS);
        const int64_t grid = (int64_t)per_sm * num_sms;
        if ((int64_t)ntiles * nbands > grid) continue;
        plan->L = L;
        plan->LS = LS;
        plan->ntiles = ntiles;
        plan->nseg = (int)nbands;
        plan->grid = (int)grid;
        plan->threads = pers::THREADS;
        plan->smem = smem;
        return cudaSuccess;
    }
    return cudaErrorNotSupported;
}

cudaError_t launch_persist(const PersistPlan& plan, const Geometry& g, int N, int iters, const float* kc, float lam,
                           float step, float* X, float* Z, const float* T, const float* chat, const float* dx,
                           const float* A1y, float* out, unsigned* resid, float* maps, unsigned* flags,
                           unsigned long long* bar, unsigned long long bar_base, unsigned epoch0, cudaStream_t s) {
    pers::Params p = {};
    p.X = X;
    p.Z = Z;
    p.T = T;
    p.chat = chat;
    p.dx = dx;
    p.A1y = A1y;
    p.out = out;
    p.resid = resid;
    p.maps = maps;
    p.flags = flags;
    p.bar = bar;
    p.bar_base = bar_base;
    p.pitch = g.pitch;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.N = N;
    p.iters = iters;
    p.ntiles = plan.ntiles;
    p.nseg = plan.nseg;
    p.epoch0 = epoch0;
    for (int i = 0; i < 4; ++i) p.kc[i] = i < N ? kc[i] : 0.f;
    p.lam = lam;
    p.step = step;
    p.timers = persist_timers();
    const void* fn = pers::kernel_for(plan.L, plan.LS);
    if (!fn) return cudaErrorInvalidValue;
    void* args[] = {&p};
    cudaError_t e =
        cudaLaunchCooperativeKernel(fn, dim3((unsigned)plan.grid), dim3((unsigned)plan.threads), args, plan.smem, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace dts
