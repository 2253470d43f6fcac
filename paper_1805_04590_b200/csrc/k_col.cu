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
// columns, so every access of a warp is one 128-B row segment.  The image is cut
// into work items = (column tile of 32 columns) x (band of HB rows).  A
// cooperative, persistent grid walks the items band-minor; each item is staged
// on chip with TMA (one box + mbarrier per Ls-row segment) and read from HBM
// exactly once:
//   1. fold each segment into an affine map; warp-shuffle scan over segments;
//   2. re-sweep with the band's causal carry c kept SYMBOLIC (y = y0 + y1 c) and
//      fold the anticausal map symbolically too, giving the band's 5-tuple
//          y_bottom = A c + B,    z_top = z0 + S c + Q e
//      (e = anticausal carry from below) -- the same tuple the multi-GPU row-band
//      exchange sends over NCCL;
//   3. publish the tuple (global memory + release flag), wait for the other
//      bands of the tile (acquire), and compose the exact carries (c, e) of this
//      band from all tuples -- no serial carry chain between bands;
//   4. finish in shared memory and leave by TMA tensor stores (FILTER) or a
//      vectorised, fully parallel update / support loop.
// Co-residency of the whole grid (required by the flag waits) is guaranteed by
// the cooperative launch; items are walked in order, so every wait is on an
// item already owned by a resident CTA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dts_device.cuh"
#include "dts_launch.h"

namespace dts {

constexpr int TW = 32;  // columns per tile (one warp)
constexpr int LS = 32;  // rows per segment (one warp), held in registers

struct ColParams {
    float* x;        // planar state (FILTER/UPDATE input; FILTER output through tm_x)
    const float* d;  // d_y (halo row)
    float* support;  // SUPPORT: S, multiplied in place by s_y
    UpdateArgs upd;
    float* tuples;           // [ntiles][nb][NTUP][TW] band tuples
    float* carries;          // [ntiles][nb][2][NV][TW] composed (c, e) per band
    unsigned int* counters;  // [ntiles] arrivals (reset to 0 by the last arriver)
    unsigned int* flags;     // [ntiles], == epoch when the tile's carries are released
    int64_t plane, pitch;
    int H, W, HB, S, Ls, nb, ntiles, nitems;
    unsigned int epoch;
    float kc;
    // row-band (multi-GPU) support: this grid covers rows [0, H) of a taller image
    int phase;                // PHASE_FULL, PHASE_TUPLE (emit the rank tuple only), PHASE_APPLY
    int halo_below;           // d row H exists: coefficient linking row H-1 to the next rank's row 0
    const float* ext;         // APPLY: [ntiles][2][NV][TW] causal carry in (top), anticausal carry in (bottom)
    float* rank_tuples;       // TUPLE: [ntiles][NTUP][TW] aggregate tuple of rows [0, H)
};

// tuple components: A, B[NV], Q, Z0[NV], Sresp  (NTUP = 2 NV + 3)
__host__ __device__ constexpr int ntup(int NV) { return 2 * NV + 3; }

struct ColSmem {  // float offsets into dynamic shared memory
    int xs, As, segF, segR, totF, totR, tup, cj, carry, bars;
    size_t bytes;
};

__host__ __device__ inline ColSmem col_smem_layout(int NV, int HB, int S, int nb) {
    ColSmem L;
    int o = 0;
    L.xs = o;
    o += NV * HB * TW;  // samples -> y0 -> y -> zbar (SUPPORT: P, then s_y)
    L.As = o;
    o += (HB + 1) * TW;  // coefficients + halo row
    L.segF = o;
    o += (NV + 1) * S * (TW + 1);
    L.segR = o;
    o += (NV + 2) * S * (TW + 1);
    L.totF = o;
    o += (NV + 1) * TW;
    L.totR = o;
    o += (NV + 2) * TW;
    L.tup = o;  // the tile's band tuples, staged from global [nb][NTUP][TW]
    o += nb * (2 * NV + 3) * TW;
    L.cj = o;  // causal carries of every band of the tile [nb][NV][TW] (TUPLE: [nb][NV+1][TW])
    o += nb * (NV + 1) * TW;
    L.carry = o;  // c[NV][TW], e[NV][TW]
    o += 2 * NV * TW;
    o = (o + 1) & ~1;  // 8-B alignment for the mbarriers
    L.bars = o;
    o += 2 * S;
    L.bytes = (size_t)o * sizeof(float);
    return L;
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp-shuffle scan across the S segment maps of column `cc` (lane = segment).
// Components: P (comp 0) and NB offsets (comps 1..NB).  Forward: exclusive
// prefix written back in place; reverse: exclusive suffix (segments below,
// applied bottom-up).  Lanes >= S are identity.  The total goes to tot[comp][cc].
template <int NB, bool REV>
__device__ __forceinline__ void seg_scan(float* seg, int S, int cc, float* tot) {
    const int lane = threadIdx.x & 31;
    Aff<NB> v = aff_identity<NB>();
    if (lane < S) {
        v.P = seg[(0 * S + lane) * (TW + 1) + cc];
#pragma unroll
        for (int k = 0; k < NB; ++k) v.B[k] = seg[((1 + k) * S + lane) * (TW + 1) + cc];
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Aff<NB> e;
        e.P = REV ? __shfl_down_sync(FULL, v.P, off) : __shfl_up_sync(FULL, v.P, off);
#pragma unroll
        for (int k = 0; k < NB; ++k) e.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], off) : __shfl_up_sync(FULL, v.B[k], off);
        const bool take = REV ? (lane + off < 32) : (lane >= off);
        if (take) v = aff_compose(e, v);
    }
    Aff<NB> ex;
    ex.P = REV ? __shfl_down_sync(FULL, v.P, 1) : __shfl_up_sync(FULL, v.P, 1);
#pragma unroll
    for (int k = 0; k < NB; ++k) ex.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], 1) : __shfl_up_sync(FULL, v.B[k], 1);
    if (REV ? lane == 31 : lane == 0) ex = aff_identity<NB>();
    if (lane < S) {
        seg[(0 * S + lane) * (TW + 1) + cc] = ex.P;
#pragma unroll
        for (int k = 0; k < NB; ++k) seg[((1 + k) * S + lane) * (TW + 1) + cc] = ex.B[k];
    }
    if (lane == (REV ? 0 : 31)) {
        tot[0 * TW + cc] = v.P;
#pragma unroll
        for (int k = 0; k < NB; ++k) tot[(1 + k) * TW + cc] = v.B[k];
    }
}

template <int CT, int MODE>
__global__ void __launch_bounds__(256)
    k_col_pass(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_d, const ColParams p) {
    constexpr int NV = (MODE == MODE_SUPPORT) ? 1 : CT;
    constexpr bool HASX = MODE != MODE_SUPPORT;
    constexpr int NT = ntup(NV);
    extern __shared__ __align__(128) float smem[];
    const int HB = p.HB, S = p.S, nb = p.nb;
    const ColSmem L = col_smem_layout(NV, HB, S, nb);
    float* xs = smem + L.xs;  // TMA landing zone: samples of the NEXT item
    float* As = smem + L.As;  // TMA landing zone: d_y of the next item (+ halo coefficient)
    float* segF = smem + L.segF;
    float* segR = smem + L.segR;
    float* totF = smem + L.totF;
    float* totR = smem + L.totR;
    float* tupS = smem + L.tup;
    float* cj = smem + L.cj;
    float* cc_ = smem + L.carry;  // c[NV][TW]
    float* ec_ = cc_ + NV * TW;   // e[NV][TW]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);

    const int c = threadIdx.x & 31;
    const int s = threadIdx.x >> 5;  // segment == warp
    const int lo = s * LS;

    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tm_d);
        if (HASX) tma_prefetch_desc(&tm_x);
    }
    __syncthreads();

    // Coefficient of row `row` as seen by the anticausal step of row-1 (R4, R20): the
    // filter coefficient inside [0, H); at row H the link to the rank below (halo) or 0
    // at the image bottom; pass-through (1) on padding rows beyond, so that a carry
    // entering at the band bottom reaches row H-1 unchanged.  The causal step of a
    // padding row uses 1 as well (see causal()).
    auto coefA = [&](int row, bool colok, float dv) -> float {
        if (!colok) return 0.f;
        if (row < p.H) return coef_from_d(dv, p.kc);
        if (row == p.H) return p.halo_below ? coef_from_d(dv, p.kc) : 0.f;
        return 1.f;
    };

    // issue the TMA loads of `item` (thread 0) and its halo coefficient (warp 0)
    auto stage_in = [&](int item) {
        const int t = item / nb;
        const int b = item - t * nb;
        const int col0 = t * TW;
        const int r0 = b * HB;
        if (threadIdx.x == 0) {
            const uint32_t box = (uint32_t)(LS * TW * sizeof(float));
            for (int q = 0; q < S; ++q) {
                const int rq = r0 + q * LS;
                const uint32_t bytes = rq < p.H ? box * (1 + (HASX ? NV : 0)) : 0u;
                mbar_arrive_expect_tx(&bars[q], bytes);
                if (bytes) {
                    tma_load_2d(As + q * LS * TW, &tm_d, col0, rq, &bars[q]);
                    if constexpr (HASX) {
#pragma unroll
                        for (int v = 0; v < NV; ++v)
                            tma_load_3d(xs + (v * HB + q * LS) * TW, &tm_x, col0, rq, v, &bars[q]);
                    }
                }
            }
        }
        if (s == 0) {
            const int rh = r0 + HB;
            const int cl = col0 + c;
            const bool inb = cl < p.W && (rh < p.H || (rh == p.H && p.halo_below));
            As[HB * TW + c] = coefA(rh, cl < p.W, inb ? p.d[(int64_t)rh * p.pitch + cl] : 0.f);
        }
    };

    if (blockIdx.x < p.nitems) stage_in(blockIdx.x);

    int k = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, ++k) {
        const int t = item / nb;
        const int b = item - t * nb;
        const int col0 = t * TW;
        const int col = col0 + c;
        const bool colok = col < p.W;
        const int r0 = b * HB;

        // ---- 1. this thread's LS rows -> registers (d -> A, invalid samples zeroed) ----
        mbar_wait(&bars[s], (uint32_t)(k & 1));
        float a[LS];
        float xv[NV][LS];
#pragma unroll
        for (int j = 0; j < LS; ++j) {
            const int rr = lo + j;
            const bool ok = colok && (r0 + rr) < p.H;
            a[j] = coefA(r0 + rr, colok, As[rr * TW + c]);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if constexpr (HASX) xv[v][j] = ok ? xs[(v * HB + rr) * TW + c] : 0.f;
                else xv[v][j] = 0.f;
            }
        }
        // causal coefficient of local row j: padding rows beyond H pass the state through
        auto causal = [&](int j) -> float { return (colok && r0 + lo + j >= p.H) ? 1.f : a[j]; };
        // causal fold
        {
            Aff<NV> m = aff_identity<NV>();
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                const float aj = causal(j);
                m.P *= aj;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) m.B[v] = fmaf(aj, m.B[v] - xv[v][j], xv[v][j]);
                    else m.B[v] = fmaf(aj, m.B[v], (colok && r0 + lo + j >= p.H) ? 0.f : 1.f);
                }
            }
            segF[(0 * S + s) * (TW + 1) + c] = m.P;
#pragma unroll
            for (int v = 0; v < NV; ++v) segF[((1 + v) * S + s) * (TW + 1) + c] = m.B[v];
        }
        __syncthreads();
        for (int cc = s; cc < TW; cc += S) seg_scan<NV, false>(segF, S, cc, totF);
        // coefficient between this segment's last row and the next row (every box has landed:
        // each warp waited on its own barrier before the barrier above)
        float anext;
        {
            const int rn = r0 + lo + LS;
            if (s + 1 < S) anext = coefA(rn, colok, As[(lo + LS) * TW + c]);
            else anext = As[HB * TW + c];  // halo (already a coefficient)
        }
        __syncthreads();  // (the landing zone is free from here on)
        {
            const int nxt = item + gridDim.x;
            if (nxt < p.nitems) stage_in(nxt);  // next item streams in under everything below
        }

        // ---- 2. symbolic causal apply (y0: carry 0, y1: response to carry 1) and
        //         symbolic anticausal fold:  z_lo = Q z_hi + E0 + E1 c ----
        {
            float y0[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) y0[v] = segF[((1 + v) * S + s) * (TW + 1) + c];
            float y1 = segF[(0 * S + s) * (TW + 1) + c];
            float Q = 1.f, E1 = 0.f, E0[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) E0[v] = 0.f;
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                const float an = (j + 1 < LS) ? a[j + 1] : anext;
                const float aj = causal(j);
                const bool valid = !(colok && r0 + lo + j >= p.H);
                y1 *= aj;
                if constexpr (HASX) {
                    const float qb = Q * (1.f - an);
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        y0[v] = fmaf(aj, y0[v] - xv[v][j], xv[v][j]);
                        xv[v][j] = y0[v];
                        E0[v] = fmaf(qb, y0[v], E0[v]);
                    }
                    E1 = fmaf(qb, y1, E1);
                } else {
                    y0[0] = fmaf(aj, y0[0], valid ? 1.f : 0.f);
                    xv[0][j] = y0[0];
                    if (valid) E0[0] += Q;  // anticausal input is 1 on valid rows, independent of c
                }
                Q *= an;
            }
            segR[(0 * S + s) * (TW + 1) + c] = Q;
#pragma unroll
            for (int v = 0; v < NV; ++v) segR[((1 + v) * S + s) * (TW + 1) + c] = E0[v];
            segR[((1 + NV) * S + s) * (TW + 1) + c] = E1;
        }
        __syncthreads();
        for (int cc = s; cc < TW; cc += S) seg_scan<NV + 1, true>(segR, S, cc, totR);
        __syncthreads();

        // ---- 3. publish this band's tuple; the LAST band of the tile to arrive composes
        //         the exact carries (c_j, e_j) of every band of the tile and releases them ----
        const float* tup_tile = p.tuples + (int64_t)t * nb * NT * TW;
        float* car_tile = p.carries + (int64_t)t * nb * 2 * NV * TW;
        if (s == 0) {
            float* tb = p.tuples + ((int64_t)t * nb + b) * NT * TW;
            tb[0 * TW + c] = totF[0 * TW + c];  // A
#pragma unroll
            for (int v = 0; v < NV; ++v) tb[(1 + v) * TW + c] = totF[(1 + v) * TW + c];  // B
            tb[(1 + NV) * TW + c] = totR[0 * TW + c];                                    // Q
#pragma unroll
            for (int v = 0; v < NV; ++v) tb[(2 + NV + v) * TW + c] = totR[(1 + v) * TW + c];  // Z0
            tb[(2 + 2 * NV) * TW + c] = totR[(1 + NV) * TW + c];                                // Sresp
            __syncwarp();
            unsigned int old = 0;
            if (c == 0) {
                __threadfence();
                old = atomicAdd(p.counters + t, 1u);
            }
            old = __shfl_sync(FULL, old, 0);
            cc_[0] = __uint_as_float(old == (unsigned)(nb - 1) ? 1u : 0u);
        }
        __syncthreads();
        if (__float_as_uint(cc_[0]) == 1u) {  // last arriver (CTA-uniform)
            __threadfence();
            const int n = nb * NT * TW;  // stage all tuples of the tile, 16 loads in flight per thread
            for (int i0 = threadIdx.x; i0 < n; i0 += 16 * blockDim.x) {
                float r[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int i = i0 + u * blockDim.x;
                    r[u] = i < n ? __ldcg(tup_tile + i) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < n) tupS[i] = r[u];
                }
            }
            __syncthreads();
            if (s == 0 && p.phase == PHASE_TUPLE) {
                // aggregate tuple of all local bands, symbolic in the carries (c, e) of the
                // rank band:  c_j = Ac c + Bc (top-down), e_{j-1} = Ze + Se c + Qe e (bottom-up)
                float Ac = 1.f, Bc[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) Bc[v] = 0.f;
                for (int j = 0; j < nb; ++j) {
                    const float* tj = tupS + j * NT * TW;
                    cj[(j * (NV + 1) + 0) * TW + c] = Ac;  // park (Ac_j, Bc_j)
#pragma unroll
                    for (int v = 0; v < NV; ++v) cj[(j * (NV + 1) + 1 + v) * TW + c] = Bc[v];
                    const float A = tj[c];
#pragma unroll
                    for (int v = 0; v < NV; ++v) Bc[v] = fmaf(A, Bc[v], tj[(1 + v) * TW + c]);
                    Ac *= A;
                }
                float Ze[NV], Se = 0.f, Qe = 1.f;
#pragma unroll
                for (int v = 0; v < NV; ++v) Ze[v] = 0.f;
                for (int j = nb - 1; j >= 0; --j) {
                    const float* tj = tupS + j * NT * TW;
                    const float Qj = tj[(1 + NV) * TW + c];
                    const float Sj = tj[(2 + 2 * NV) * TW + c];
                    const float Acj = cj[(j * (NV + 1) + 0) * TW + c];
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        Ze[v] = fmaf(Qj, Ze[v], fmaf(Sj, cj[(j * (NV + 1) + 1 + v) * TW + c], tj[(2 + NV + v) * TW + c]));
                    Se = fmaf(Qj, Se, Sj * Acj);
                    Qe *= Qj;
                }
                float* rt = p.rank_tuples + (int64_t)t * NT * TW;
                rt[0 * TW + c] = Ac;
#pragma unroll
                for (int v = 0; v < NV; ++v) rt[(1 + v) * TW + c] = Bc[v];
                rt[(1 + NV) * TW + c] = Qe;
#pragma unroll
                for (int v = 0; v < NV; ++v) rt[(2 + NV + v) * TW + c] = Ze[v];
                rt[(2 + 2 * NV) * TW + c] = Se;
                __syncwarp();
                if (c == 0) p.counters[t] = 0u;  // ready for the next launch
            } else if (s == 0) {
                const float* ext = p.phase == PHASE_APPLY ? p.ext + (int64_t)t * 2 * NV * TW : nullptr;
                float cv[NV];  // causal carries c_j (c_0 = carry into the rank band, 0 on a single GPU)
#pragma unroll
                for (int v = 0; v < NV; ++v) cv[v] = ext ? ext[v * TW + c] : 0.f;
                for (int j = 0; j < nb; ++j) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        cj[(j * NV + v) * TW + c] = cv[v];
                        car_tile[((int64_t)(j * 2 + 0) * NV + v) * TW + c] = cv[v];
                    }
                    const float* tj = tupS + j * NT * TW;
                    const float A = tj[c];
#pragma unroll
                    for (int v = 0; v < NV; ++v) cv[v] = fmaf(A, cv[v], tj[(1 + v) * TW + c]);
                }
                float ev[NV];  // anticausal carries: e_{j-1} = Z0_j + Sresp_j c_j + Q_j e_j, e_last = carry in
#pragma unroll
                for (int v = 0; v < NV; ++v) ev[v] = ext ? ext[(NV + v) * TW + c] : 0.f;
                for (int j = nb - 1; j >= 0; --j) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) car_tile[((int64_t)(j * 2 + 1) * NV + v) * TW + c] = ev[v];
                    const float* tj = tupS + j * NT * TW;
                    const float Qj = tj[(1 + NV) * TW + c];
                    const float Sj = tj[(2 + 2 * NV) * TW + c];
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        ev[v] = fmaf(Qj, ev[v], fmaf(Sj, cj[(j * NV + v) * TW + c], tj[(2 + NV + v) * TW + c]));
                }
                __syncwarp();
                if (c == 0) {
                    p.counters[t] = 0u;  // ready for the next launch
                    __threadfence();
                    st_release_u32(p.flags + t, p.epoch);
                }
            }
        }
        if (p.phase == PHASE_TUPLE) {  // only the tuples were wanted
            __syncthreads();
            continue;
        }
        if (s == 0) {
            if (c == 0)
                while (ld_acquire_u32(p.flags + t) != p.epoch) __nanosleep(32);
            __syncwarp();
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                cc_[v * TW + c] = __ldcg(car_tile + ((int64_t)(b * 2 + 0) * NV + v) * TW + c);
                ec_[v * TW + c] = __ldcg(car_tile + ((int64_t)(b * 2 + 1) * NV + v) * TW + c);
            }
        }
        __syncthreads();

        // ---- 4. exact causal values y = y0 + y1 c, then anticausal apply (registers) ----
        {
            float cv[NV], z[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) cv[v] = cc_[v * TW + c];
            float y1 = segF[(0 * S + s) * (TW + 1) + c];
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                y1 *= causal(j);
#pragma unroll
                for (int v = 0; v < NV; ++v) xv[v][j] = fmaf(y1, cv[v], xv[v][j]);
            }
            const float eQ = segR[(0 * S + s) * (TW + 1) + c];
            const float eS = segR[((1 + NV) * S + s) * (TW + 1) + c];
#pragma unroll
            for (int v = 0; v < NV; ++v)
                z[v] = fmaf(eQ, ec_[v * TW + c], fmaf(eS, cv[v], segR[((1 + v) * S + s) * (TW + 1) + c]));
#pragma unroll
            for (int j = LS - 1; j >= 0; --j) {
                const float an = (j + 1 < LS) ? a[j + 1] : anext;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float yv = xv[v][j];
                    if constexpr (HASX) {
                        z[v] = fmaf(an, z[v] - yv, yv);
                        xv[v][j] = z[v];
                    } else {
                        const bool valid = !(colok && r0 + lo + j >= p.H);
                        z[v] = fmaf(an, z[v], valid ? 1.f : 0.f);
                        xv[v][j] = yv + z[v] - 1.f;  // s_y = P + Q - 1
                    }
                }
            }
        }

        // ---- 5. write-out straight from registers (a warp stores one 128-B row segment) ----
        {
            const int nrow = min(LS, p.H - (r0 + lo));
            if (colok && nrow > 0) {
                if constexpr (MODE == MODE_FILTER) {
#pragma unroll
                    for (int j = 0; j < LS; ++j)
                        if (j < nrow) {
                            const int64_t o = (int64_t)(r0 + lo + j) * p.pitch + col;
#pragma unroll
                            for (int v = 0; v < NV; ++v) p.x[v * p.plane + o] = xv[v][j];
                        }
                } else if constexpr (MODE == MODE_SUPPORT) {
#pragma unroll
                    for (int j = 0; j < LS; ++j)
                        if (j < nrow) {
                            const int64_t o = (int64_t)(r0 + lo + j) * p.pitch + col;
                            p.support[o] *= xv[0][j];
                        }
                } else {  // MODE_UPDATE: Eq. (3) with zbar = xv
#pragma unroll
                    for (int j0 = 0; j0 < LS; j0 += 8) {
                        float zo[8][NV], tv[8][NV], ch[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = j0 + u;
                            const int64_t o = (int64_t)(r0 + lo + (j < nrow ? j : 0)) * p.pitch + col;
                            ch[u] = __ldg(p.upd.chat + o);
#pragma unroll
                            for (int v = 0; v < NV; ++v) {
                                zo[u][v] = p.upd.Z[v * p.plane + o];
                                tv[u][v] = __ldg(p.upd.T + v * p.plane + o);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = j0 + u;
                            if (j < nrow) {
                                const int64_t r = r0 + lo + j;
                                const int64_t o = r * p.pitch + col;
#pragma unroll
                                for (int v = 0; v < NV; ++v) {
                                    const float g = fmaf(p.upd.lam, zo[u][v] - xv[v][j], ch[u] * (zo[u][v] - tv[u][v]));
                                    const float zn = fmaf(-p.upd.step, g, zo[u][v]);
                                    if (p.upd.out_hwc) p.upd.out_hwc[(r * p.W + col) * CT + v] = zn;
                                    else p.upd.Z[v * p.plane + o] = zn;
                                }
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();  // segF / segR / tuples are rewritten by the next item
    }
}

// Row-band exchange, second half: from the gathered rank tuples (in rank order) compute
// the carries into rank `rank`:  c_{q+1} = A_q c_q + B_q (c_0 = 0, the image top);
// e_{q-1} = Z0_q + S_q c_q + Q_q e_q (e_{P-1} = 0, the image bottom).  One thread per column.
__global__ void k_rank_compose(const float* __restrict__ g, int P, int rank, int ntiles, int NV,
                               float* __restrict__ ext) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntiles * TW) return;
    const int t = i / TW, c = i - t * TW;
    const int NT = 2 * NV + 3;
    const int64_t rstride = (int64_t)ntiles * NT * TW;  // one rank's tuples
    const float* base = g + (int64_t)t * NT * TW + c;
    for (int v = 0; v < NV; ++v) {
        float cq[64];
        float cv = 0.f;
        for (int q = 0; q < P; ++q) {
            cq[q] = cv;
            const float* tq = base + q * rstride;
            cv = fmaf(tq[0], cv, tq[(1 + v) * TW]);
        }
        float ev = 0.f;
        for (int q = P - 1; q > rank; --q) {
            const float* tq = base + q * rstride;
            ev = fmaf(tq[(1 + NV) * TW], ev, fmaf(tq[(2 + 2 * NV) * TW], cq[q], tq[(2 + NV + v) * TW]));
        }
        ext[((int64_t)t * 2 * NV + v) * TW + c] = cq[rank];
        ext[((int64_t)t * 2 * NV + NV + v) * TW + c] = ev;
    }
}

cudaError_t launch_rank_compose(const float* gathered, int P, int rank, int ntiles, int NV, float* ext,
                                cudaStream_t s) {
    if (P > 64) return cudaErrorInvalidValue;
    const int n = ntiles * TW;
    k_rank_compose<<<(n + 127) / 128, 128, 0, s>>>(gathered, P, rank, ntiles, NV, ext);
    return cudaGetLastError();
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

// rank-3 map over planar fp32 data [planes][H][pitch], box {TW, rows, 1}
static bool make_tmap3(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int64_t planes, int rows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)H, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * sizeof(float)), (cuuint64_t)(pitch * H * sizeof(float))};
    cuuint32_t box[3] = {(cuuint32_t)TW, (cuuint32_t)rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool make_tmap2(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int rows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)H};
    cuuint64_t strides[1] = {(cuuint64_t)(pitch * sizeof(float))};
    cuuint32_t box[2] = {(cuuint32_t)TW, (cuuint32_t)rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static const size_t kSmemMax = 227 * 1024;
static const int kLs = LS;

template <int CT, int MODE>
static const void* kernel_ptr() {
    return reinterpret_cast<const void*>(k_col_pass<CT, MODE>);
}

static const void* col_kernel(int Ct, int mode) {
    if (mode == MODE_SUPPORT) return kernel_ptr<1, MODE_SUPPORT>();
    switch (Ct * 4 + mode) {
        case 4 + MODE_FILTER: return kernel_ptr<1, MODE_FILTER>();
        case 8 + MODE_FILTER: return kernel_ptr<2, MODE_FILTER>();
        case 12 + MODE_FILTER: return kernel_ptr<3, MODE_FILTER>();
        case 16 + MODE_FILTER: return kernel_ptr<4, MODE_FILTER>();
        case 4 + MODE_UPDATE: return kernel_ptr<1, MODE_UPDATE>();
        case 8 + MODE_UPDATE: return kernel_ptr<2, MODE_UPDATE>();
        case 12 + MODE_UPDATE: return kernel_ptr<3, MODE_UPDATE>();
        case 16 + MODE_UPDATE: return kernel_ptr<4, MODE_UPDATE>();
    }
    return nullptr;
}

cudaError_t plan_col_pass(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan) {
    const int NV = (mode == MODE_SUPPORT) ? 1 : Ct;
    const void* fn = col_kernel(Ct, mode);
    if (!fn) return cudaErrorInvalidValue;
    // band height: S segments of kLs rows; aim for >= 2 resident CTAs per SM
    int S = (int)((g.H + kLs - 1) / kLs);
    const int Smax = NV >= 3 ? 6 : 8;
    if (S > Smax) S = Smax;
    if (S < 1) S = 1;
    const int HB = S * kLs;
    const int nb = (int)((g.H + HB - 1) / HB);
    const ColSmem L = col_smem_layout(NV, HB, S, nb);
    if (L.bytes > kSmemMax) return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem_attr(fn, L.bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, TW * S, L.bytes);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidValue;
    const int ntiles = (int)((g.W + TW - 1) / TW);
    const int64_t nitems = (int64_t)ntiles * nb;
    if (nb > per_sm * num_sms) return cudaErrorInvalidValue;  // a tile's bands must be co-resident
    int64_t grid = (int64_t)per_sm * num_sms;
    if (grid > nitems) grid = nitems;
    plan->kind = 0;
    plan->TW = TW;
    plan->CB = 1;
    plan->HB = HB;
    plan->S = S;
    plan->Ls = kLs;
    plan->nb = nb;
    plan->ntiles = ntiles;
    plan->threads = TW * S;
    plan->grid = dim3((unsigned)grid, 1, 1);
    plan->smem = L.bytes;
    plan->tuple_floats = (size_t)nitems * (ntup(4) + 2 * 4) * TW;  // tuples + carries (NV <= 4)
    plan->flag_count = (size_t)ntiles * 2;                           // flags + counters
    return cudaSuccess;
}

cudaError_t launch_col_pass(const ColPlan& plan, const Geometry& g, int Ct, int mode, float* x, const float* d,
                            float kc, const UpdateArgs* upd, float* support, const ColScratch& scr,
                            cudaStream_t s) {
    ColParams p = {};
    p.x = x;
    p.d = d;
    p.support = support;
    if (upd) p.upd = *upd;
    p.tuples = scr.tuples;
    p.carries = scr.tuples + (size_t)plan.ntiles * plan.nb * ntup(4) * TW;
    p.flags = scr.flags;
    p.counters = scr.flags + plan.ntiles;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.HB = plan.HB;
    p.S = plan.S;
    p.Ls = plan.Ls;
    p.nb = plan.nb;
    p.ntiles = plan.ntiles;
    p.nitems = plan.ntiles * plan.nb;
    p.epoch = scr.epoch;
    p.kc = kc;
    p.phase = scr.phase;
    p.halo_below = scr.halo_below;
    p.ext = scr.ext;
    p.rank_tuples = scr.rank_tuples;
    CUtensorMap tx, td;
    if (!make_tmap2(&td, d, g.pitch, g.H + (scr.halo_below ? 1 : 0), plan.Ls)) return cudaErrorInvalidValue;
    if (mode != MODE_SUPPORT) {
        if (!make_tmap3(&tx, x, g.pitch, g.H, Ct, plan.Ls)) return cudaErrorInvalidValue;
    } else {
        tx = td;  // unused
    }
    const void* fn = col_kernel(Ct, mode);
    if (!fn) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = plan.grid;
    cfg.blockDim = dim3((unsigned)plan.threads, 1, 1);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the in-kernel tuple waits
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&tx, &td, &p};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace dts
