// k_col2p.cu -- K3: column pass as a two-phase decoupled band-tuple scan with an L2 lag
// (sm_100a).  High occupancy, no on-chip holding: latency is hidden by resident CTAs.
//
// Recurrence (R4-R6), per column, A = a_i^{d_y}:
//     causal      y[r] = (1 - A[r]) x[r] + A[r] y[r-1]              (A[0] = 0: d_y[0] = +inf)
//     anticausal  z[r] = (1 - A[r+1]) y[r] + A[r+1] z[r+1]          (A[H] = 0: d_y[H] = +inf)
//
// Work item = (tile of 64 columns) x (band of HB = NW*LR rows).  Lane l of a warp owns
// columns 2l, 2l+1 (float2: packed FFMA2 math, 256-B coalesced row segments), warp w owns
// rows [w LR, (w+1) LR) of the band.  Items are numbered tile-major; CTA c of the
// persistent grid (all CTAs co-resident, several per SM) walks positions i = c, c+G, ...
// and at each position runs
//   PHASE 1 of item i: load its x and d rows (HBM; they stay in L2), fold each warp's rows
//     into a segment 5-tuple  y_out = A c + B,  z_top = Z0 + S c + Q e  (c: causal state
//     from above, e: anticausal state from below), compose the band tuple and publish it
//     (release + arrival counter);
//   PHASE 2 of item i - LAG: wait for its tile's carries (almost always already out), load
//     the rows again (L2 hits: LAG items ~ 40 MB of L2), refold, derive the warp's own
//     carries, sweep causal forward and anticausal backward, store.
//   The CTA whose band arrives last at a tile composes the exact carries (c_b, e_b) of all
//     bands of the tile (8 warps, one round trip of tuple loads) and releases the tile.
// HBM traffic is the algorithmic 12 B/pixel (x, d in; X out) as long as the lagged
// re-read hits L2; ncu's dram bytes per launch check it (profiles/).
// Deadlock freedom: phase 1 never waits; a phase 2 at position i waits only on tiles
// whose bands sit at positions <= i - LAG + nb - 1 < i, all of them processed in phase 1
// by resident CTAs before any of them can block.
#include "dts_device.cuh"
#include "dts_launch.h"

#include <cstdio>
#include <cstdlib>

namespace dts {
namespace col2p {

constexpr int TW = 64;  // columns per tile
constexpr int NW = 8;   // warps per CTA
constexpr int NTHREADS = NW * 32;

__host__ __device__ constexpr int ntup(int NV) { return 3 + 2 * NV; }  // A, Q, S, B[NV], Z0[NV]
__host__ __device__ constexpr int lrows(int NV) { return NV == 1 ? 16 : 8; }
__host__ __device__ constexpr int maxb(int NV) { return NV == 1 ? 10 : 5; }  // bands per warp in a composition

struct Params {
    float* x;        // planar state, in place
    const float* d;  // d_y, rows 0..H (row H: +inf at the image bottom)
    float* tup;      // [ntiles][nb][NT][TW] band tuples
    float* car;      // [ntiles][nb][2 NV][TW] composed carries (c, e)
    unsigned int* counters;  // [ntiles] band arrivals (reset by the composer)
    unsigned int* flags;     // [ntiles] == epoch once the tile's carries are out
    int64_t plane, pitch;
    int H, W, HB, nb, ntiles, nitems, lag;
    unsigned int epoch;
    float kc;
};

// ---- packed fp32 helpers (FFMA2 / FMUL2 / FADD2) ----------------------------------------
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
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
__device__ __forceinline__ float2 ldg2(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ float2 ldcg2(const float* p) { return __ldcg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ void stcg2(float* p, float2 v) { __stcg(reinterpret_cast<float2*>(p), v); }
// L2 eviction-priority policies: phase 1 keeps its rows (they are read again by phase 2),
// phase 2's re-read and the output stream leave first
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float2 ldh2(const float* p, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void sth2(float* p, float2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
template <int NV>
__device__ __forceinline__ void store_tup(float* base, const Tup<NV>& t) {
    sts2(base + 0 * TW, t.A);
    sts2(base + 1 * TW, t.Q);
    sts2(base + 2 * TW, t.S);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        sts2(base + (3 + v) * TW, t.B[v]);
        sts2(base + (3 + NV + v) * TW, t.Z0[v]);
    }
}

// The warp's rows of item (t, b): coefficients A and samples x into registers (rows
// beyond H: A = 1, x = 0, except the link row H whose d is +inf; columns beyond the pitch:
// A = 0, x = 0), the link coefficient below the warp's last row, and the segment tuple.
template <int NV, int LR>
__device__ __forceinline__ Tup<NV> load_fold(const Params& p, int t, int b, float2 (&a)[LR], float2 (&xv)[NV][LR],
                                             float2& ab, uint64_t pol) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int col = t * TW + 2 * lane;
    const bool colok = col < p.pitch;
    const int r0 = b * p.HB + w * LR;
    const float nkc = -p.kc;
    const float* dp = p.d + (int64_t)r0 * p.pitch + col;
    const float* xp = p.x + (int64_t)r0 * p.pitch + col;
    if (colok && r0 + LR < p.H) {  // fast path: every row (and the link row) inside the image
#pragma unroll
        for (int j = 0; j < LR; ++j) {
            a[j] = ldh2(dp + j * p.pitch, pol);
#pragma unroll
            for (int v = 0; v < NV; ++v) xv[v][j] = ldh2(xp + v * p.plane + j * p.pitch, pol);
        }
        ab = ldh2(dp + LR * p.pitch, pol);
    } else {
#pragma unroll
        for (int j = 0; j < LR; ++j) {
            const int r = r0 + j;
            a[j] = !colok ? f2(__int_as_float(0x7f800000)) : (r <= p.H ? ldg2(dp + j * p.pitch) : f2(0.f));
#pragma unroll
            for (int v = 0; v < NV; ++v)
                xv[v][j] = (colok && r < p.H) ? *reinterpret_cast<const float2*>(xp + v * p.plane + j * p.pitch) : f2(0.f);
        }
        const int rl = r0 + LR;
        ab = !colok ? f2(__int_as_float(0x7f800000)) : (rl <= p.H ? ldg2(dp + LR * p.pitch) : f2(0.f));
    }
#pragma unroll
    for (int j = 0; j < LR; ++j) a[j] = coef2(a[j], nkc);
    ab = coef2(ab, nkc);
    Tup<NV> m;
    float2 P = f2(1.f), q = f2(1.f), S = f2(0.f), y0[NV], Z0[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) y0[v] = Z0[v] = f2(0.f);
#pragma unroll
    for (int j = 0; j < LR; ++j) {
        if (j > 0) {  // close row j-1: its anticausal link is A[j]
            const float2 wgt = mul2(q, sub2(f2(1.f), a[j]));
#pragma unroll
            for (int v = 0; v < NV; ++v) Z0[v] = fma2(wgt, y0[v], Z0[v]);
            S = fma2(wgt, P, S);
            q = mul2(q, a[j]);
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) y0[v] = rstep(a[j], y0[v], xv[v][j]);
        P = mul2(P, a[j]);
    }
    {
        const float2 wgt = mul2(q, sub2(f2(1.f), ab));
#pragma unroll
        for (int v = 0; v < NV; ++v) Z0[v] = fma2(wgt, y0[v], Z0[v]);
        S = fma2(wgt, P, S);
        q = mul2(q, ab);
    }
    m.A = P;
    m.Q = q;
    m.S = S;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        m.B[v] = y0[v];
        m.Z0[v] = Z0[v];
    }
    return m;
}

// Cooperative (whole CTA) composition of tile t's carries from its nb band tuples.
template <int NV>
__device__ __noinline__ void compose_tile(const float* tup, float* car, unsigned int* counters, unsigned int* flags,
                                          int nb, unsigned int epoch, int t, float* agg) {
    constexpr int NT = ntup(NV);
    constexpr int MB = maxb(NV);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, cl = 2 * lane;
    __threadfence();  // acquire side of the arrival counter
    const int per = (nb + NW - 1) / NW;
    const int b0 = w * per;
    const int nmine = max(0, min(per, nb - b0));
    Tup<NV> T[MB];
    const float* tt = tup + ((size_t)t * nb * NT) * TW + cl;
#pragma unroll
    for (int u = 0; u < MB; ++u) {
        if (u < nmine) {
            const float* tb = tt + (size_t)(b0 + u) * NT * TW;
            T[u].A = ldcg2(tb);
            T[u].Q = ldcg2(tb + 1 * TW);
            T[u].S = ldcg2(tb + 2 * TW);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                T[u].B[v] = ldcg2(tb + (3 + v) * TW);
                T[u].Z0[v] = ldcg2(tb + (3 + NV + v) * TW);
            }
        }
    }
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
    __syncthreads();
    float2 c[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) c[v] = f2(0.f);
    for (int k = 0; k < w; ++k) {
        const float* ak = agg + k * (1 + NV) * TW + cl;
        const float2 A = lds2(ak);
#pragma unroll
        for (int v = 0; v < NV; ++v) c[v] = fma2(A, c[v], lds2(ak + (1 + v) * TW));
    }
    float* cc = car + ((size_t)t * nb * 2 * NV) * TW + cl;
#pragma unroll
    for (int u = 0; u < MB; ++u) {  // causal carries; K = Z0 + S c kept in Z0
        if (u < nmine) {
            float* cb = cc + (size_t)(b0 + u) * 2 * NV * TW;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                stcg2(cb + v * TW, c[v]);
                T[u].Z0[v] = fma2(T[u].S, c[v], T[u].Z0[v]);
                c[v] = fma2(T[u].A, c[v], T[u].B[v]);
            }
        }
    }
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
    __syncthreads();
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
            float* cb = cc + (size_t)(b0 + u) * 2 * NV * TW;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                stcg2(cb + (NV + v) * TW, e[v]);
                e[v] = fma2(T[u].Q, e[v], T[u].Z0[v]);
            }
        }
    }
    __threadfence();
    __syncthreads();  // every carry stored and fenced; agg free again
    if (threadIdx.x == 0) {
        counters[t] = 0u;
        st_release(&flags[t], epoch);
    }
}

template <int NV>
__global__ void __launch_bounds__(NTHREADS, 2) k_col_2p(const Params p) {
    constexpr int NT = ntup(NV);
    constexpr int LR = lrows(NV);
    extern __shared__ __align__(16) float dsm[];
    float* scratch0 = dsm;                      // chunk tuples, phase 1
    float* scratch1 = dsm + NW * NT * TW;       // chunk tuples, phase 2
    float* agg = dsm + 2 * NW * NT * TW;        // composition aggregates
    int* s_compose_p = reinterpret_cast<int*>(agg + 2 * NW * (1 + NV) * TW);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, cl = 2 * lane;
    const int G = gridDim.x;
    const int nb = p.nb;

    for (int i = blockIdx.x; i < p.nitems + p.lag; i += G) {
        // ---------------- PHASE 1 of item i ----------------
        unsigned int old = 0;
        int ptile = -1;
        if (i < p.nitems) {
            const int t = i / nb, b = i - t * nb;
            float2 a[LR], xv[NV][LR], ab;
            const Tup<NV> m = load_fold<NV, LR>(p, t, b, a, xv, ab, pol_last());
            float* sc = scratch0;
            store_tup<NV>(sc + w * NT * TW + cl, m);
            __syncthreads();
            if (w == 0) {  // band tuple -> global, then count the arrival
                Tup<NV> acc = load_tup<NV>(sc + cl);
                for (int c = 1; c < NW; ++c) acc = compose<NV>(acc, load_tup<NV>(sc + c * NT * TW + cl));
                float* gt = p.tup + ((size_t)(t * nb + b) * NT) * TW + cl;
                stcg2(gt + 0 * TW, acc.A);
                stcg2(gt + 1 * TW, acc.Q);
                stcg2(gt + 2 * TW, acc.S);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    stcg2(gt + (3 + v) * TW, acc.B[v]);
                    stcg2(gt + (3 + NV + v) * TW, acc.Z0[v]);
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) old = atomicAdd(&p.counters[t], 1u);  // result used after phase 2
                ptile = t;
            }
        }
        // ---------------- PHASE 2 of item i - lag ----------------
        const int i2 = i - p.lag;
        if (i2 >= 0) {
            const int t = i2 / nb, b = i2 - t * nb;
            // carries of the tile (released long ago in the steady state)
            if (lane == 0) {
                while (ld_acquire(&p.flags[t]) != p.epoch) __nanosleep(64);
            }
            __syncwarp();
            (void)ld_acquire(&p.flags[t]);
            const float* cb = p.car + ((size_t)(t * nb + b) * 2 * NV) * TW + cl;
            float2 cc[NV], ee[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                cc[v] = ldcg2(cb + v * TW);
                ee[v] = ldcg2(cb + (NV + v) * TW);
            }
            float2 a[LR], xv[NV][LR], ab;
            const Tup<NV> m = load_fold<NV, LR>(p, t, b, a, xv, ab, pol_first());
            float* sc = scratch1;
            store_tup<NV>(sc + w * NT * TW + cl, m);
            __syncthreads();
            // causal entry of this warp: chunks above; anticausal entry: chunks below
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
            float2 sZ0[NV], sS = f2(0.f), sQ = f2(1.f);
#pragma unroll
            for (int v = 0; v < NV; ++v) sZ0[v] = f2(0.f);
            for (int c = NW - 1; c > w; --c) {
                const Tup<NV> U = load_tup<NV>(sc + c * NT * TW + cl);
#pragma unroll
                for (int v = 0; v < NV; ++v) sZ0[v] = fma2(U.Q, fma2(sS, U.B[v], sZ0[v]), U.Z0[v]);
                sS = fma2(mul2(U.Q, sS), U.A, U.S);
                sQ = mul2(U.Q, sQ);
            }
            float2 y[NV], z[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                y[v] = fma2(Apre, cc[v], Bpre[v]);  // causal state entering the warp's rows
                // anticausal state entering from below: the chunks below see the causal
                // state leaving this warp's rows, y_out = A y + B
                const float2 yo = fma2(m.A, y[v], m.B[v]);
                z[v] = fma2(sQ, ee[v], fma2(sS, yo, sZ0[v]));
            }
#pragma unroll
            for (int j = 0; j < LR; ++j) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    y[v] = rstep(a[j], y[v], xv[v][j]);
                    xv[v][j] = y[v];
                }
            }
            const int col = t * TW + cl;
            const int r0 = b * p.HB + w * LR;
            float* o = p.x + (int64_t)r0 * p.pitch + col;
            if (col + 1 < p.W && r0 + LR <= p.H) {
                const uint64_t pf = pol_first();
#pragma unroll
                for (int j = LR - 1; j >= 0; --j) {
                    const float2 an = (j + 1 < LR) ? a[j + 1] : ab;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        z[v] = rstep(an, z[v], xv[v][j]);
                        sth2(o + v * p.plane + j * p.pitch, z[v], pf);
                    }
                }
            } else {
                const bool ok2 = col + 1 < p.W, ok1 = col < p.W;
#pragma unroll
                for (int j = LR - 1; j >= 0; --j) {
                    const float2 an = (j + 1 < LR) ? a[j + 1] : ab;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        z[v] = rstep(an, z[v], xv[v][j]);
                        if (r0 + j < p.H) {
                            if (ok2) *reinterpret_cast<float2*>(o + v * p.plane + j * p.pitch) = z[v];
                            else if (ok1) o[v * p.plane + j * p.pitch] = z[v].x;
                        }
                    }
                }
            }
        }
        // ---------------- composition, if this CTA's band arrived last ----------------
        if (threadIdx.x == 0) *s_compose_p = (ptile >= 0 && old == (unsigned)(nb - 1)) ? ptile : -1;
        __syncthreads();
        const int ct = *s_compose_p;
        if (ct >= 0) compose_tile<NV>(p.tup, p.car, p.counters, p.flags, nb, p.epoch, ct, agg);
        __syncthreads();  // s_compose / scratch reuse
    }
}

}  // namespace col2p

static const void* col2p_kernel(int Ct) {
    switch (Ct) {
        case 1: return reinterpret_cast<const void*>(col2p::k_col_2p<1>);
        case 2: return reinterpret_cast<const void*>(col2p::k_col_2p<2>);
        case 3: return reinterpret_cast<const void*>(col2p::k_col_2p<3>);
    }
    return nullptr;
}

static size_t col2p_smem(int NV) {
    return (size_t)(2 * col2p::NW * col2p::ntup(NV) * col2p::TW + 2 * col2p::NW * (1 + NV) * col2p::TW + 4) *
           sizeof(float);
}

cudaError_t plan_col_2p(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan) {
    if (mode != MODE_FILTER || Ct < 1 || Ct > 3) return cudaErrorNotSupported;
    const void* fn = col2p_kernel(Ct);
    const int LR = col2p::lrows(Ct);
    const int HB = col2p::NW * LR;
    const int ntiles = (int)((g.W + col2p::TW - 1) / col2p::TW);
    const int64_t nb = (g.H + HB - 1) / HB;
    if (nb > (int64_t)col2p::NW * col2p::maxb(Ct)) return cudaErrorNotSupported;  // composition capacity
    const size_t smem = col2p_smem(Ct);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, col2p::NTHREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorNotSupported;
    const int64_t nitems = nb * ntiles;
    int64_t G = (int64_t)num_sms * per_sm;
    if (G > nitems) G = nitems;
    plan->kind = 3;
    plan->TW = col2p::TW;
    plan->CB = 1;
    plan->HB = HB;
    plan->S = col2p::NW;
    plan->Ls = LR;
    plan->nb = (int)nb;
    plan->ntiles = ntiles;
    plan->threads = col2p::NTHREADS;
    plan->grid = dim3((unsigned)G, 1, 1);
    plan->smem = smem;
    plan->tuple_floats = (size_t)ntiles * nb * (col2p::ntup(Ct) + 2 * Ct) * col2p::TW;
    plan->flag_count = 2 * (size_t)ntiles;
    return cudaSuccess;
}

cudaError_t launch_col_2p(const ColPlan& plan, const Geometry& g, int Ct, float* x, const float* d, float kc,
                          const ColScratch& scr, cudaStream_t s) {
    col2p::Params p = {};
    p.x = x;
    p.d = d;
    p.tup = scr.tuples;
    p.car = scr.tuples + (size_t)plan.ntiles * plan.nb * col2p::ntup(Ct) * col2p::TW;
    p.counters = scr.flags;
    p.flags = scr.flags + plan.ntiles;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.HB = plan.HB;
    p.nb = plan.nb;
    p.ntiles = plan.ntiles;
    p.nitems = plan.nb * plan.ntiles;
    // lag: a whole tile plus two grid widths of items -> the tile is complete and composed
    // long before its phase 2; ~LAG x 64 KB of x/d stay live in L2
    static const int lag_env = std::getenv("DTS_COL2P_LAG") ? std::atoi(std::getenv("DTS_COL2P_LAG")) : 0;
    const int G = (int)plan.grid.x;
    p.lag = lag_env > 0 ? lag_env : plan.nb + G;
    p.epoch = scr.epoch;
    p.kc = kc;
    const void* fn = col2p_kernel(Ct);
    if (!fn) return cudaErrorInvalidValue;
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel(fn, plan.grid, dim3((unsigned)plan.threads, 1, 1), args, plan.smem, s);
}

}  // namespace dts
