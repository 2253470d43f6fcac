// k_colv.cu -- K3: streaming column pass (sm_100a).  Decoupled band-tuple scan whose
// lagged work items live in TENSOR MEMORY; no atomics, no blocking acquires.
//
// Recurrence (R4-R6), per column, A = a_i^{d_y}:
//     causal      y[r] = (1 - A[r]) x[r] + A[r] y[r-1]              (A[0] = 0: d_y[0] = +inf)
//     anticausal  z[r] = (1 - A[r+1]) y[r] + A[r+1] z[r+1]          (A[H] = 0: d_y[H] = +inf)
//
// Work item = (tile of 64 columns) x (band of HB = NW*LR rows); lane l of a warp owns
// columns 2l, 2l+1 (float2 everywhere: FFMA2 math, 256-B row segments), warp w owns rows
// [w LR, (w+1) LR) of the band.  Item i = (tile i / nb, band i % nb); CTA g of the
// persistent grid (one per SM, co-resident) takes items g, g+G, g+2G, ...
//
// Step j of a CTA (8 warps):
//   PHASE 1 of item j: wait for its TMA tensor loads (x: HB rows, d_y: HB+1 rows -- the
//     last links the band to the next), fold each warp's rows into a segment 5-tuple
//         y_out = A c + B,   z_top = Z0 + S c + Q e
//     (c: causal state entering from above, e: anticausal state from below), park x and
//     A in TMEM (tcgen05.st), release the landing slot (warp 0 refills it by TMA with
//     item j+2), compose the chunk tuples into the band tuple and publish it as 64-bit
//     {value, epoch} words (single-copy atomic: visible and self-validating, no fence).
//   PHASE 2 of item j-3: carries (c_b, e_b) arrive as 64-bit {value, epoch} words (one
//     relaxed load, issued at the start of the step), x and A come back from TMEM
//     (tcgen05.ld); causal sweep forward into registers, anticausal sweep backward, stores.
//   The CTA that holds the last band of a tile composes that tile's carries: its 8 warps
//     load the tagged band tuples (one L2 round trip; retried later if any word is stale),
//     fold them in registers, exchange 8 partial aggregates through shared memory and
//     store every band's tagged carries.
// TMEM holds NREG = 4 items per warp (x and A of 16 rows x 2 columns = 64 columns; the
// warp's prefix/suffix maps of the item wait in shared memory), so
// phase 2 runs 3 steps (~7 us) behind phase 1 and the composition is off the critical
// path.  Every pixel is read from HBM once and written once per pass.
// Deadlock freedom: a CTA waiting for carries keeps attempting its pending compositions;
// a composition only waits for band tuples of items no later than one step ahead, and
// nb <= G (one item of a CTA per tile).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dts_device.cuh"
#include "dts_launch.h"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace dts {
namespace colv {

constexpr int TW = 64;     // columns per tile
constexpr int NSLOT = 2;   // TMA landing slots
constexpr int NREG = 4;    // TMEM item regions per consumer warp (lag = NREG - 1 steps)
constexpr int NW = 8;      // warps: TMEM lane quarter w % 4, column half w / 4 (256 columns each);
                          // two per SMSP, so each may hold up to 255 registers
constexpr int NTHREADS = NW * 32;
constexpr int NDBG = 8;

__host__ __device__ constexpr int ntup(int NV) { return 3 + 2 * NV; }  // A, Q, S, B[NV], Z0[NV]
__host__ __device__ constexpr int lrows(int NV) { return NV == 1 ? 16 : (NV == 2 ? 8 : 4); }  // (NV+1)*2*LR <= 64 TMEM columns
__host__ __device__ constexpr int ninfo(int NV) { return 4 + 2 * NV; }  // float2 words of a warp's Info
__host__ __device__ constexpr int maxb(int NV) { return NV == 1 ? 10 : 5; }  // bands per warp in a composition

struct Params {
    float* x;        // planar state, in place
    const float* d;  // d_y, rows 0..H (row H: +inf at the image bottom, or the halo)
    unsigned long long* tup;    // [ntiles][nb][NT][TW] band tuples as {value, epoch} words
    unsigned long long* car;    // [ntiles][nb][2 NV][TW] carries (c, e) as {value, epoch}
    int64_t plane, pitch;
    int H, W, HB, nb, ntiles, nitems;
    unsigned int epoch;
    float kc;
    unsigned long long* dbg;  // optional phase timers [G][NDBG] (DTS_COLV_DEBUG)
};

struct Layout {
    size_t slot, scratch, agg, info, vote, bars, bytes;
};
__host__ __device__ inline Layout layout(int NV, int HB) {
    const int NT = ntup(NV);
    Layout L;
    size_t o = 0;  // floats
    L.slot = o;
    o += (size_t)NSLOT * (NV * HB + HB + 1) * TW;
    L.scratch = o;  // chunk tuples, double-buffered by step parity
    o += (size_t)2 * NW * NT * TW;
    L.agg = o;  // composition aggregates (causal A,B[NV]; anticausal Q,K[NV])
    o += (size_t)2 * NW * (1 + NV) * TW;
    L.info = o;  // per (region, warp): the warp's Info between phase 1 and phase 2
    o += (size_t)NREG * NW * ninfo(NV) * 2 * TW / 2;
    L.vote = o;  // u32 [2][NW] votes, tmem base
    o += 2 * NW + 2;
    o = (o + 1) & ~(size_t)1;
    L.bars = o;  // u64 full[NSLOT]
    o += 2 * NSLOT;
    L.bytes = o * sizeof(float);
    return L;
}

// ---- packed fp32 helpers (FFMA2 / FMUL2 / FADD2 on sm_100a) ----------------------------
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// one recurrence step  s <- a (s - v) + v  ==  (1 - a) v + a s
__device__ __forceinline__ float2 rstep(float2 a, float2 s, float2 v) { return fma2(a, sub2(s, v), v); }

__device__ __forceinline__ float2 coef2(float2 d, float nkc) {
    const float2 t = mul2(d, f2(nkc));
    float2 y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(t.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(t.y));
    return y;
}

__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void sts2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
__device__ __forceinline__ float2 ldcg2(const float* p) { return __ldcg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ void stcg2(float* p, float2 v) { __stcg(reinterpret_cast<float2*>(p), v); }

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cta_sync() { __syncthreads(); }
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// tagged 64-bit words {value bits, epoch}: single-copy atomic, so value and tag agree
__device__ __forceinline__ void st_tag(unsigned long long* p, float v, unsigned int tag) {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tag(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ long long clk() { return clock64(); }

// ---- tensor memory ------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc512(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst_smem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 8 consecutive TMEM columns of this thread's lane <-> 8 registers (32x32b shape)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, float2 a, float2 b, float2 c, float2 d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y), "f"(d.x), "f"(d.y)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float2& a, float2& b, float2& c, float2& d) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y), "=f"(c.x), "=f"(c.y), "=f"(d.x), "=f"(d.y)
                 : "r"(taddr)
                 : "memory");
}

template <int NV>
struct Tup {
    float2 A, Q, S, B[NV], Z0[NV];
};
// U above L  ->  the combined segment
template <int NV>
__device__ __forceinline__ Tup<NV> compose(const Tup<NV>& U, const Tup<NV>& L) {
    Tup<NV> r;
    r.A = mul2(L.A, U.A);
    r.Q = mul2(U.Q, L.Q);
    r.S = fma2(mul2(U.Q, L.S), U.A, U.S);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        r.B[v] = fma2(L.A, U.B[v], L.B[v]);
        r.Z0[v] = fma2(U.Q, fma2(L.S, U.B[v], L.Z0[v]), U.Z0[v]);
    }
    return r;
}
template <int NV>
__device__ __forceinline__ Tup<NV> load_tup(const float* base) {  // [NT][TW] at this lane's column
    Tup<NV> t;
    t.A = lds2(base + 0 * TW);
    t.Q = lds2(base + 1 * TW);
    t.S = lds2(base + 2 * TW);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        t.B[v] = lds2(base + (3 + v) * TW);
        t.Z0[v] = lds2(base + (3 + NV + v) * TW);
    }
    return t;
}

// What a warp keeps between phase 1 and phase 2 of an item:
//     c_w = Apre c_b + Bpre,   e_w = E0 + Ec c_b + Ee e_b,   ab = link coefficient below
template <int NV>
struct Info {
    float2 Apre, Ec, Ee, ab, Bpre[NV], E0[NV];
};

// Collective over the CTA (every warp calls it): compose tile t's carries if all of its band
// tuples are up.  Rare (about once per tile), so it is kept out of line: its registers do
// not burden the streaming loop.
template <int NV>
__device__ __noinline__ bool try_compose(unsigned long long* tup, unsigned long long* car, int nb, unsigned int epoch,
                                         int t, float* agg, volatile uint32_t* vote) {
    constexpr int NT = ntup(NV);
    constexpr int MB = maxb(NV);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cl = 2 * lane;
        const int per = (nb + NW - 1) / NW;
    const int b0 = w * per;
    const int nmine = max(0, min(per, nb - b0));
    // tagged band tuples of my bands: all words must carry this launch's epoch
    Tup<NV> T[MB];
    bool ok = true;
    const unsigned long long* tt = tup + ((size_t)t * nb * NT) * TW + cl;
    auto ldv = [&](const unsigned long long* q) -> float2 {
        const unsigned long long a = ld_tag(q), b = ld_tag(q + 1);
        ok = ok && (unsigned int)(a >> 32) == epoch && (unsigned int)(b >> 32) == epoch;
        return make_float2(__uint_as_float((uint32_t)a), __uint_as_float((uint32_t)b));
    };
#pragma unroll
    for (int u = 0; u < MB; ++u) {
        if (u < nmine) {
            const unsigned long long* tb = tt + (size_t)(b0 + u) * NT * TW;
            T[u].A = ldv(tb);
            T[u].Q = ldv(tb + 1 * TW);
            T[u].S = ldv(tb + 2 * TW);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                T[u].B[v] = ldv(tb + (3 + v) * TW);
                T[u].Z0[v] = ldv(tb + (3 + NV + v) * TW);
            }
        }
    }
    ok = __all_sync(FULL, ok);
    if (lane == 0) vote[NW + w] = ok ? 1u : 0u;
    __syncthreads();
    bool all = true;
#pragma unroll
    for (int k = 0; k < NW; ++k) all = all && vote[NW + k] != 0u;
    __syncthreads();
    if (!all) return false;
    // causal aggregate of my bands
    float2 Ag = f2(1.f), Bg[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Bg[v] = f2(0.f);
#pragma unroll
    for (int u = 0; u < MB; ++u) {
        if (u < nmine) {
#pragma unroll
            for (int v = 0; v < NV; ++v) Bg[v] = fma2(T[u].A, Bg[v], T[u].B[v]);
            Ag = mul2(T[u].A, Ag);
        }
    }
    float* ag = agg + w * (1 + NV) * TW + cl;
    sts2(ag, Ag);
#pragma unroll
    for (int v = 0; v < NV; ++v) sts2(ag + (1 + v) * TW, Bg[v]);
    cta_sync();
    float2 c[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) c[v] = f2(0.f);
    for (int k = 0; k < w; ++k) {
        const float* ak = agg + k * (1 + NV) * TW + cl;
        const float2 A = lds2(ak);
#pragma unroll
        for (int v = 0; v < NV; ++v) c[v] = fma2(A, c[v], lds2(ak + (1 + v) * TW));
    }
    unsigned long long* cc = car + ((size_t)t * nb * 2 * NV) * TW + cl;
    // walk my bands: causal carries out, K = Z0 + S c (kept in Z0)
#pragma unroll
    for (int u = 0; u < MB; ++u) {
        if (u < nmine) {
            unsigned long long* cb = cc + (size_t)(b0 + u) * 2 * NV * TW;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                st_tag(cb + v * TW, c[v].x, epoch);
                st_tag(cb + v * TW + 1, c[v].y, epoch);
                T[u].Z0[v] = fma2(T[u].S, c[v], T[u].Z0[v]);
                c[v] = fma2(T[u].A, c[v], T[u].B[v]);
            }
        }
    }
    // anticausal aggregate of my bands (bottom-up): e_top = K + Q e_in
    float2 Qg = f2(1.f), Kg[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Kg[v] = f2(0.f);
#pragma unroll
    for (int u = MB - 1; u >= 0; --u) {
        if (u < nmine) {
#pragma unroll
            for (int v = 0; v < NV; ++v) Kg[v] = fma2(T[u].Q, Kg[v], T[u].Z0[v]);
            Qg = mul2(T[u].Q, Qg);
        }
    }
    float* ag2 = agg + (NW + w) * (1 + NV) * TW + cl;
    sts2(ag2, Qg);
#pragma unroll
    for (int v = 0; v < NV; ++v) sts2(ag2 + (1 + v) * TW, Kg[v]);
    cta_sync();
    float2 e[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) e[v] = f2(0.f);
    for (int k = NW - 1; k > w; --k) {
        const float* ak = agg + (NW + k) * (1 + NV) * TW + cl;
        const float2 Q = lds2(ak);
#pragma unroll
        for (int v = 0; v < NV; ++v) e[v] = fma2(Q, e[v], lds2(ak + (1 + v) * TW));
    }
#pragma unroll
    for (int u = MB - 1; u >= 0; --u) {
        if (u < nmine) {
            unsigned long long* cb = cc + (size_t)(b0 + u) * 2 * NV * TW;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                st_tag(cb + (NV + v) * TW, e[v].x, epoch);
                st_tag(cb + (NV + v) * TW + 1, e[v].y, epoch);
                e[v] = fma2(T[u].Q, e[v], T[u].Z0[v]);
            }
        }
    }
    cta_sync();  // agg is reused by the next composition
    return true;
}

template <int NV>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_col_v(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_d, const Params p) {
    constexpr int NT = ntup(NV);
    constexpr int LR = lrows(NV);
    constexpr int MB = maxb(NV);
    constexpr int NCW = 4 * NV;  // tagged carry words per lane: c[v].xy, e[v].xy
    constexpr int NI = ninfo(NV);
    static_assert((NV + 1) * 2 * LR <= 64 && LR % 4 == 0, "TMEM region holds 64 columns, written 4 rows at a time");
    extern __shared__ __align__(128) float smem[];
    const int HB = p.HB, nb = p.nb;
    const Layout Lo = layout(NV, HB);
    const size_t SF = (size_t)(NV * HB + HB + 1) * TW;
    float* scratch = smem + Lo.scratch;
    float* agg = smem + Lo.agg;
    volatile uint32_t* vote = reinterpret_cast<volatile uint32_t*>(smem + Lo.vote);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lo.bars);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x;
    const int nloc = (p.nitems - (int)blockIdx.x + G - 1) / G;
    const int cl = 2 * lane;
    const unsigned int epoch = p.epoch;

    auto item_tile = [&](int j) { return ((int)blockIdx.x + j * G) / nb; };
    auto item_band = [&](int j) { return ((int)blockIdx.x + j * G) % nb; };
    auto issue = [&](int j) {  // thread 0: TMA tensor loads of item j into its landing slot
        const int s = j % NSLOT;
        const int t = item_tile(j), b = item_band(j);
        float* xs = smem + Lo.slot + s * SF;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(SF * sizeof(float)));
        tma_load_2d(xs + NV * HB * TW, &tm_d, t * TW, b * HB, &full[s]);
#pragma unroll
        for (int v = 0; v < NV; ++v) tma_load_3d(xs + v * HB * TW, &tm_x, t * TW, b * HB, v, &full[s]);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NSLOT; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    if (w == 0) tmem_alloc512(const_cast<uint32_t*>(vote + 2 * NW));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = vote[2 * NW];
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tm_d);
        tma_prefetch_desc(&tm_x);
        for (int j = 0; j < NSLOT && j < nloc; ++j) issue(j);
    }

    const int rw = w * LR;
    const uint32_t taddr = tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(256 * (w >> 2));
    const float nkc = -p.kc;
    int natt = 0, ncomp = 0;
    unsigned int c_tma = 0, c_vote = 0, c_all = 0, c_att = 0;  // cycle counters (DTS_COLV_DEBUG)
    const unsigned int c_start = (unsigned int)clock();

    // tiles whose last band this CTA holds, awaiting composition (warp-uniform queue)
    int pend0 = 0, pend1 = 0, pend2 = 0, pend3 = 0, npend = 0;
    auto attempt = [&]() -> bool {
        ++natt;
        const unsigned int c0 = (unsigned int)clock();
        const bool okc = try_compose<NV>(p.tup, p.car, nb, epoch, pend0, agg, vote);
        c_att += (unsigned int)clock() - c0;
        if (!okc) return false;
        ++ncomp;
        pend0 = pend1;
        pend1 = pend2;
        pend2 = pend3;
        --npend;
        return true;
    };
    float* infos = smem + Lo.info;  // [NREG][NW][NI][TW] float2 words at this lane's column
    for (int j = 0; j < nloc + NREG - 1; ++j) {
        const int i = j - (NREG - 1);
        // ---- carries of item i (tagged), in flight during phase 1 ----
        unsigned long long cw[NCW];
        const unsigned long long* cwp = nullptr;
        if (i >= 0) {
            cwp = p.car + ((size_t)(item_tile(i) * nb + item_band(i)) * 2 * NV) * TW + cl;
#pragma unroll
            for (int k = 0; k < 2 * NV; ++k) {
                cw[2 * k] = ld_tag(cwp + k * TW);
                cw[2 * k + 1] = ld_tag(cwp + k * TW + 1);
            }
        }
        // ---------------- PHASE 1 of item j ----------------
        if (j < nloc) {
            const int s = j % NSLOT, r = j % NREG;
            const float* xs = smem + Lo.slot + s * SF;
            const float* ds = xs + NV * HB * TW;
            {
                const unsigned int c0 = (unsigned int)clock();
                mbar_wait(&full[s], (uint32_t)((j / NSLOT) & 1));
                c_tma += (unsigned int)clock() - c0;
            }
            const float2 ab = coef2(lds2(ds + (rw + LR) * TW + cl), nkc);
            float2 av[LR], xv[NV][LR];
            float2 y0[NV], Z0[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) y0[v] = Z0[v] = f2(0.f);
            float2 P = f2(1.f), q = f2(1.f), S = f2(0.f);
#pragma unroll
            for (int jj = 0; jj < LR; ++jj) {
                const float2 a = coef2(lds2(ds + (rw + jj) * TW + cl), nkc);
                av[jj] = a;
                if (jj > 0) {  // close row jj-1: its anticausal link is A[jj]
                    const float2 wgt = mul2(q, sub2(f2(1.f), a));
#pragma unroll
                    for (int v = 0; v < NV; ++v) Z0[v] = fma2(wgt, y0[v], Z0[v]);
                    S = fma2(wgt, P, S);
                    q = mul2(q, a);
                }
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    xv[v][jj] = lds2(xs + (v * HB + rw + jj) * TW + cl);
                    y0[v] = rstep(a, y0[v], xv[v][jj]);
                }
                P = mul2(P, a);
            }
            {
                const float2 wgt = mul2(q, sub2(f2(1.f), ab));
#pragma unroll
                for (int v = 0; v < NV; ++v) Z0[v] = fma2(wgt, y0[v], Z0[v]);
                S = fma2(wgt, P, S);
                q = mul2(q, ab);
            }
            // TMEM region r: columns [0, 2LR) hold A of the warp's rows, [2LR(1+v), 2LR(2+v)) x[v]
#pragma unroll
            for (int g = 0; g < LR; g += 4) {
                tmem_st8(taddr + 64 * r + 2 * g, av[g], av[g + 1], av[g + 2], av[g + 3]);
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    tmem_st8(taddr + 64 * r + 2 * LR * (1 + v) + 2 * g, xv[v][g], xv[v][g + 1], xv[v][g + 2],
                             xv[v][g + 3]);
            }

            float* sc = scratch + (j & 1) * NW * NT * TW;
            float* my = sc + w * NT * TW + cl;
            sts2(my + 0 * TW, P);
            sts2(my + 1 * TW, q);
            sts2(my + 2 * TW, S);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                sts2(my + (3 + v) * TW, y0[v]);
                sts2(my + (3 + NV + v) * TW, Z0[v]);
            }
            tmem_wait_st();
            cta_sync();  // chunk tuples of item j visible; landing slot s consumed by every warp
            if (threadIdx.x == 0 && j + NSLOT < nloc) issue(j + NSLOT);

            Info<NV> in;
            in.ab = ab;
            float2 Apre = f2(1.f), Bpre[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) Bpre[v] = f2(0.f);
            for (int c = 0; c < w; ++c) {
                const float* tc = sc + c * NT * TW + cl;
                const float2 Ac = lds2(tc);
#pragma unroll
                for (int v = 0; v < NV; ++v) Bpre[v] = fma2(Ac, Bpre[v], lds2(tc + (3 + v) * TW));
                Apre = mul2(Ac, Apre);
            }
            in.Apre = Apre;
#pragma unroll
            for (int v = 0; v < NV; ++v) in.Bpre[v] = Bpre[v];
            const float2 A1 = mul2(P, Apre);
            float2 B1[NV], sZ0[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                B1[v] = fma2(P, Bpre[v], y0[v]);
                sZ0[v] = f2(0.f);
            }
            float2 sS = f2(0.f), sQ = f2(1.f);
            for (int c = NW - 1; c > w; --c) {
                const Tup<NV> U = load_tup<NV>(sc + c * NT * TW + cl);
#pragma unroll
                for (int v = 0; v < NV; ++v) sZ0[v] = fma2(U.Q, fma2(sS, U.B[v], sZ0[v]), U.Z0[v]);
                sS = fma2(mul2(U.Q, sS), U.A, U.S);
                sQ = mul2(U.Q, sQ);
            }
            in.Ec = mul2(sS, A1);
            in.Ee = sQ;
#pragma unroll
            for (int v = 0; v < NV; ++v) in.E0[v] = fma2(sS, B1[v], sZ0[v]);
            {
                float* ip = infos + ((size_t)(r * NW + w) * NI) * TW + cl;
                sts2(ip + 0 * TW, in.Apre);
                sts2(ip + 1 * TW, in.Ec);
                sts2(ip + 2 * TW, in.Ee);
                sts2(ip + 3 * TW, in.ab);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    sts2(ip + (4 + v) * TW, in.Bpre[v]);
                    sts2(ip + (4 + NV + v) * TW, in.E0[v]);
                }
            }

            const int t = item_tile(j), b = item_band(j);
            if (w == 0) {  // band tuple -> global memory as tagged words (visible as soon as stored)
                Tup<NV> acc = load_tup<NV>(sc + cl);
                for (int c = 1; c < NW; ++c) acc = compose<NV>(acc, load_tup<NV>(sc + c * NT * TW + cl));
                unsigned long long* gt = p.tup + ((size_t)(t * nb + b) * NT) * TW + cl;
                auto stv = [&](unsigned long long* q, float2 v) {
                    st_tag(q, v.x, epoch);
                    st_tag(q + 1, v.y, epoch);
                };
                stv(gt + 0 * TW, acc.A);
                stv(gt + 1 * TW, acc.Q);
                stv(gt + 2 * TW, acc.S);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    stv(gt + (3 + v) * TW, acc.B[v]);
                    stv(gt + (3 + NV + v) * TW, acc.Z0[v]);
                }
            }
            if (b == nb - 1) {
                if (npend == 0) pend0 = t;
                else if (npend == 1) pend1 = t;
                else if (npend == 2) pend2 = t;
                else pend3 = t;
                ++npend;
            }
        }
        // ---------------- PHASE 2 of item i = j-3 ----------------
        if (i >= 0) {
            const int r = i % NREG;
            const unsigned int c0 = (unsigned int)clock();
            for (;;) {  // collective: carries complete for every warp?
                bool ok = true;
#pragma unroll
                for (int k = 0; k < NCW; ++k) ok = ok && (unsigned int)(cw[k] >> 32) == epoch;
                ok = __all_sync(FULL, ok);
                if (lane == 0) vote[w] = ok ? 1u : 0u;
                cta_sync();
                bool all = true;
#pragma unroll
                for (int k = 0; k < NW; ++k) all = all && vote[k] != 0u;
                cta_sync();
                if (all) break;
                if (npend) {
                    attempt();
                } else {
                    __nanosleep(256);
                }
#pragma unroll
                for (int k = 0; k < 2 * NV; ++k) {
                    cw[2 * k] = ld_tag(cwp + k * TW);
                    cw[2 * k + 1] = ld_tag(cwp + k * TW + 1);
                }
            }
            c_vote += (unsigned int)clock() - c0;
            Info<NV> in;
            {
                const float* ip = infos + ((size_t)(r * NW + w) * NI) * TW + cl;
                in.Apre = lds2(ip + 0 * TW);
                in.Ec = lds2(ip + 1 * TW);
                in.Ee = lds2(ip + 2 * TW);
                in.ab = lds2(ip + 3 * TW);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    in.Bpre[v] = lds2(ip + (4 + v) * TW);
                    in.E0[v] = lds2(ip + (4 + NV + v) * TW);
                }
            }
            float2 y[NV], z[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float2 c = make_float2(__uint_as_float((uint32_t)cw[2 * v]), __uint_as_float((uint32_t)cw[2 * v + 1]));
                const float2 e = make_float2(__uint_as_float((uint32_t)cw[2 * NV + 2 * v]),
                                             __uint_as_float((uint32_t)cw[2 * NV + 2 * v + 1]));
                y[v] = fma2(in.Apre, c, in.Bpre[v]);
                z[v] = fma2(in.Ee, e, fma2(in.Ec, c, in.E0[v]));
            }
            float2 av[LR];
            float2 yv[NV][LR];
#pragma unroll
            for (int g = 0; g < LR; g += 4) {
                tmem_ld8(taddr + 64 * r + 2 * g, av[g], av[g + 1], av[g + 2], av[g + 3]);
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    tmem_ld8(taddr + 64 * r + 2 * LR * (1 + v) + 2 * g, yv[v][g], yv[v][g + 1], yv[v][g + 2],
                             yv[v][g + 3]);
            }
            tmem_wait_ld();
#pragma unroll
            for (int jj = 0; jj < LR; ++jj) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    y[v] = rstep(av[jj], y[v], yv[v][jj]);  // x -> y in place
                    yv[v][jj] = y[v];
                }
            }
            const int t = item_tile(i), b = item_band(i);
            const int col = t * TW + cl;
            const int r0 = b * HB + rw;
            const bool ok2 = col + 1 < p.W, ok1 = col < p.W;
#pragma unroll
            for (int jj = LR - 1; jj >= 0; --jj) {
                const float2 an = (jj + 1 < LR) ? av[jj + 1] : in.ab;
                const int row = r0 + jj;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    z[v] = rstep(an, z[v], yv[v][jj]);
                    if (row < p.H) {
                        float* o = p.x + v * p.plane + (int64_t)row * p.pitch + col;
                        if (ok2) *reinterpret_cast<float2*>(o) = z[v];
                        else if (ok1) o[0] = z[v].x;
                    }
                }
            }
        }
        // ---- opportunistic composition of a pending tile ----
        if (npend) attempt();
    }
    while (npend) {  // compositions still owed to other CTAs
        if (!attempt()) __nanosleep(256);
    }
    if (p.dbg && w == 0 && lane == 0) {
        c_all = (unsigned int)clock() - c_start;
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 0], (unsigned long long)c_tma);
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 1], (unsigned long long)c_vote);
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 2], (unsigned long long)c_att);
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 5], (unsigned long long)c_all);
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 3], (unsigned long long)ncomp);
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 4], (unsigned long long)natt);
        atomicAdd(&p.dbg[blockIdx.x * NDBG + 7], (unsigned long long)nloc);
    }
    tc_fence_before();
    __syncthreads();
    if (w == 0) {
        tc_fence_after();
        tmem_dealloc512(tbase);
    }
}

}  // namespace colv

// ---------------------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 colv_encoder() {
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

// planes of `rows` x pitch floats, `planes` of them `plane` floats apart; box 64 x box_rows
static bool colv_tmap(CUtensorMap* m, const void* base, int64_t pitch, int64_t rows, int64_t plane, int64_t planes,
                      int box_rows, cuuint32_t rank) {
    auto enc = colv_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * sizeof(float)), (cuuint64_t)(plane * sizeof(float))};
    cuuint32_t box[3] = {(cuuint32_t)colv::TW, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static const void* colv_kernel(int Ct) {
    switch (Ct) {
        case 1: return reinterpret_cast<const void*>(colv::k_col_v<1>);
        case 2: return reinterpret_cast<const void*>(colv::k_col_v<2>);
        case 3: return reinterpret_cast<const void*>(colv::k_col_v<3>);
    }
    return nullptr;
}

cudaError_t plan_col_stream(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan) {
    if (mode != MODE_FILTER || Ct < 1 || Ct > 3) return cudaErrorNotSupported;
    const void* fn = colv_kernel(Ct);
    if (!fn) return cudaErrorNotSupported;
    const int LR = colv::lrows(Ct);
    const int HB = colv::NW * LR;
    const colv::Layout L = colv::layout(Ct, HB);
    if (L.bytes > 227 * 1024) return cudaErrorNotSupported;
    const int ntiles = (int)((g.W + colv::TW - 1) / colv::TW);
    const int64_t nb = (g.H + HB - 1) / HB;
    const int64_t nitems = nb * ntiles;
    if (nb > (int64_t)colv::NW * colv::maxb(Ct)) return cudaErrorNotSupported;  // composition capacity
    const int G = (int)(nitems < num_sms ? nitems : num_sms);
    if (nb > G) return cudaErrorNotSupported;  // one item of a CTA per tile
    static const bool dbg = std::getenv("DTS_DEBUG") != nullptr;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes);
    if (e != cudaSuccess) {
        if (dbg) std::fprintf(stderr, "plan_col_stream: smem attribute: %s\n", cudaGetErrorString(e));
        return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, colv::NTHREADS, L.bytes);
    if (e != cudaSuccess || per_sm < 1) {
        if (dbg) std::fprintf(stderr, "plan_col_stream: occupancy %d (%s)\n", per_sm, cudaGetErrorString(e));
        return e != cudaSuccess ? e : cudaErrorNotSupported;
    }
    plan->kind = 2;
    plan->TW = colv::TW;
    plan->CB = 1;
    plan->HB = HB;
    plan->S = colv::NW;
    plan->Ls = LR;
    plan->nb = (int)nb;
    plan->ntiles = ntiles;
    plan->threads = colv::NTHREADS;
    plan->grid = dim3((unsigned)G, 1, 1);
    plan->smem = L.bytes;
    // tagged band tuples and carries ({value, epoch} 64-bit words) in the zero-initialised
    // flag words: a stale or never-written word can never carry the current epoch
    plan->tuple_floats = 1;
    plan->flag_count = (size_t)ntiles * nb * (colv::ntup(Ct) + 2 * Ct) * colv::TW * 2;
    return cudaSuccess;
}

cudaError_t launch_col_stream(const ColPlan& plan, const Geometry& g, int Ct, int mode, float* x, const float* d,
                              float kc, const UpdateArgs* upd, const ColScratch& scr, cudaStream_t s) {
    (void)upd;
    if (mode != MODE_FILTER) return cudaErrorInvalidValue;
    colv::Params p = {};
    p.x = x;
    p.d = d;
    p.tup = reinterpret_cast<unsigned long long*>(scr.flags);
    p.car = p.tup + (size_t)plan.ntiles * plan.nb * colv::ntup(Ct) * colv::TW;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.HB = plan.HB;
    p.nb = plan.nb;
    p.ntiles = plan.ntiles;
    p.nitems = plan.nb * plan.ntiles;
    p.epoch = scr.epoch;
    p.kc = kc;
    CUtensorMap tx, td;
    if (!colv_tmap(&td, d, g.pitch, g.H + 1, g.plane, 1, plan.HB + 1, 2)) return cudaErrorInvalidValue;
    if (!colv_tmap(&tx, x, g.pitch, g.H, g.plane, Ct, plan.HB, 3)) return cudaErrorInvalidValue;
    const void* fn = colv_kernel(Ct);
    if (!fn) return cudaErrorInvalidValue;
    static const bool debug = std::getenv("DTS_COLV_DEBUG") != nullptr;
    unsigned long long* dbg = nullptr;
    const size_t nd = (size_t)plan.grid.x * colv::NDBG;
    if (debug) {
        cudaMalloc(&dbg, nd * sizeof(unsigned long long));
        cudaMemsetAsync(dbg, 0, nd * sizeof(unsigned long long), s);
        p.dbg = dbg;
    }
    void* args[] = {&tx, &td, &p};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, plan.grid, dim3((unsigned)plan.threads, 1, 1), args, plan.smem, s);
    if (debug) {
        std::vector<unsigned long long> h(nd);
        cudaMemcpyAsync(h.data(), dbg, nd * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        cudaFree(dbg);
        double tot[colv::NDBG] = {0};
        for (size_t i = 0; i < nd; ++i) tot[i % colv::NDBG] += (double)h[i];
        const double G = plan.grid.x;
        std::fprintf(stderr,
                     "colv Ct %d HB %d nb %d G %u: per CTA [kcycles] all %.1f tma-wait %.1f carry-wait %.1f "
                     "compose %.1f | compositions %.2f attempts %.2f items %.1f\n",
                     Ct, plan.HB, plan.nb, plan.grid.x, tot[5] / G / 1e3, tot[0] / G / 1e3, tot[1] / G / 1e3,
                     tot[2] / G / 1e3, tot[3] / G, tot[4] / G, tot[7] / G);
    }
    return e;
}

}  // namespace dts
