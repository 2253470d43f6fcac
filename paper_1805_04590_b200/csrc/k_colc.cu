// k_colc.cu -- K3 fast path: column pass with the column tile held by a
// thread-block CLUSTER (sm_100a), persistent over tiles, TMA-prefetching the next tile.
//
// Same recurrence as k_col.cu (R4-R7), FILTER and SUPPORT modes (+ the
// row-band TUPLE mode); the Eq. (3) step runs in the streaming update kernel or the next
// iteration's first row pass (DESIGN.md section 12 records why the fused write-out lost).  Layout of the work: a column tile is 32 columns x H rows; CTA
// b of a cluster of CB CTAs owns rows [b*HB, (b+1)*HB); inside the CTA, warp s owns
// rows [s*LS, (s+1)*LS) and lane c owns column c, holding its LS samples and
// coefficients in REGISTERS.  Per tile:
//   wait TMA boxes -> registers; the landing zone is immediately refilled with the
//   NEXT tile (TMA), so HBM streams while this tile computes;
//   causal fold -> warp-shuffle segment scan -> band totals exchanged through
//   distributed shared memory (DSMEM) after a cluster barrier -> exact causal apply
//   with the anticausal map folded on the fly -> second DSMEM exchange -> exact
//   anticausal apply -> stores straight from registers (one 128-B row segment per
//   warp instruction).
// Each pixel is read from HBM once and written once per pass; the carries between
// bands never leave the chip.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dts_device.cuh"
#include "dts_launch.h"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace dts {

namespace colc {

constexpr int TW = 32;  // columns per tile (one warp)
constexpr int LS = 32;  // rows per warp segment (registers)

struct Params {
    float* x;        // planar state (in; FILTER: out)
    const float* d;  // d_y
    float* support;  // SUPPORT: receives s_y (the solve multiplies it into S in the prologue)
    float* sedge;    // row strips (nullable): [strip][2][CT][ntc * 32] outputs at each strip's last / first row
    UpdateArgs upd;
    int64_t plane, pitch;
    int H, W, HB, S, CB, ntiles;
    int HS, ntc;  // row strips (single-GPU FILTER): strip height, column tiles per strip (HS = H: one strip)
    float kc;
    int nsq;  // < 0: d holds distances (a = 2^(-kc d)); >= 0: d holds A1, a = A1^(2^nsq)
    int pdl_early;  // trigger the dependent launch at the start (option pdl = 2) instead of the end
};

struct Smem {
    int land_x, land_d, segF, segR, totC, totA, remC, remA, carry, bars;
    size_t bytes;
};

__host__ __device__ inline Smem layout(int NV, int HB, int S) {
    Smem L;
    int o = 0;
    L.land_x = o;
    o += NV * HB * TW;
    L.land_d = o;
    o += HB * TW;
    L.segF = o;
    o += (NV + 1) * S * (TW + 1);
    L.segR = o;
    o += (NV + 1) * S * (TW + 1);
    L.totC = o;  // band totals read by the other CTAs of the cluster (DSMEM)
    o += (NV + 1) * TW;
    L.totA = o;
    o += (NV + 1) * TW;
    L.remC = o;  // band totals pushed by the bands above (st.async) [16][NV+1][TW]
    o += 16 * (NV + 1) * TW;
    L.remA = o;  // band totals pushed by the bands below
    o += 16 * (NV + 1) * TW;
    L.carry = o;
    o += NV * TW;
    o = (o + 1) & ~1;
    L.bars = o;
    o += 2 * S + 4;  // S TMA barriers + 2 exchange barriers
    L.bytes = (size_t)o * sizeof(float);
    return L;
}

// Shuffle scan of the S segment maps of column cc (lane = segment), exclusive
// results written back, total -> tot.  Lanes >= S are identity.
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
        if (REV ? (lane + off < 32) : (lane >= off)) v = aff_compose(e, v);
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

// Two columns per warp when S <= 16: lanes 0-15 scan the S segment maps of column cA,
// lanes 16-31 those of column cB (width-16 shuffles); otherwise as seg_scan.
template <int NB, bool REV>
__device__ __forceinline__ void seg_scan2(float* seg, int S, int cA, int cB, float* tot) {
    const int lane = threadIdx.x & 31;
    const int sl = lane & 15;
    const int cc = lane < 16 ? cA : cB;
    Aff<NB> v = aff_identity<NB>();
    if (sl < S) {
        v.P = seg[(0 * S + sl) * (TW + 1) + cc];
#pragma unroll
        for (int k = 0; k < NB; ++k) v.B[k] = seg[((1 + k) * S + sl) * (TW + 1) + cc];
    }
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        Aff<NB> e;
        e.P = REV ? __shfl_down_sync(FULL, v.P, off, 16) : __shfl_up_sync(FULL, v.P, off, 16);
#pragma unroll
        for (int k = 0; k < NB; ++k)
            e.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], off, 16) : __shfl_up_sync(FULL, v.B[k], off, 16);
        if (REV ? (sl + off < 16) : (sl >= off)) v = aff_compose(e, v);
    }
    Aff<NB> ex;
    ex.P = REV ? __shfl_down_sync(FULL, v.P, 1, 16) : __shfl_up_sync(FULL, v.P, 1, 16);
#pragma unroll
    for (int k = 0; k < NB; ++k)
        ex.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], 1, 16) : __shfl_up_sync(FULL, v.B[k], 1, 16);
    if (REV ? sl == 15 : sl == 0) ex = aff_identity<NB>();
    if (sl < S) {
        seg[(0 * S + sl) * (TW + 1) + cc] = ex.P;
#pragma unroll
        for (int k = 0; k < NB; ++k) seg[((1 + k) * S + sl) * (TW + 1) + cc] = ex.B[k];
    }
    if (sl == (REV ? 0 : 15)) {
        tot[0 * TW + cc] = v.P;
#pragma unroll
        for (int k = 0; k < NB; ++k) tot[(1 + k) * TW + cc] = v.B[k];
    }
}

// Grouped segment scan: GR lane groups per column, 32 / GR columns per warp, so GR warps cover
// the 32 columns of a tile.  Lane = (column cl = lane % (32 / GR), group g = lane / (32 / GR));
// group g owns m = ceil(S / GR) consecutive segments: it folds them serially (loads first, all
// independent), the GR group totals of a column are scanned with log2(GR) shuffle steps, and
// each group writes its segments' exclusive prefixes while re-folding them.  GR = 4 at NB = 3:
// ~125 warp instructions for 8 columns against ~140 per column for the one-column-per-warp
// shuffle scan (seg_scan).  REV scans from the last segment.  Same results as seg_scan up to the
// association order of the compositions.
template <int NB, bool REV, int GR>
__device__ __forceinline__ void seg_scan_grp(float* seg, int S, int w, float* tot) {
    constexpr int CW = 32 / GR;  // columns per warp
    const int lane = threadIdx.x & 31;
    const int cl = lane % CW, g = lane / CW;
    const int cc = w * CW + cl;
    const int m = (S + GR - 1) / GR;
    const int lo = min(S, g * m), hi = min(S, lo + m);
    constexpr int MMAX = (24 + GR - 1) / GR;  // S <= 24
    // local fold (upstream first: ascending, or descending for REV)
    Aff<NB> v = aff_identity<NB>();
#pragma unroll
    for (int q = 0; q < MMAX; ++q) {
        const int sg = REV ? hi - 1 - q : lo + q;
        if (q < hi - lo) {
            Aff<NB> e;
            e.P = seg[(0 * S + sg) * (TW + 1) + cc];
#pragma unroll
            for (int k = 0; k < NB; ++k) e.B[k] = seg[((1 + k) * S + sg) * (TW + 1) + cc];
            v = aff_compose(v, e);
        }
    }
    // inclusive scan over the GR groups of a column (upstream groups: lower g, or higher for REV)
#pragma unroll
    for (int off = CW; off < 32; off <<= 1) {
        Aff<NB> e;
        e.P = REV ? __shfl_down_sync(FULL, v.P, off) : __shfl_up_sync(FULL, v.P, off);
#pragma unroll
        for (int k = 0; k < NB; ++k) e.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], off) : __shfl_up_sync(FULL, v.B[k], off);
        if (REV ? (lane + off < 32) : (lane >= off)) v = aff_compose(e, v);
    }
    if (g == (REV ? 0 : GR - 1)) {
        tot[0 * TW + cc] = v.P;
#pragma unroll
        for (int k = 0; k < NB; ++k) tot[(1 + k) * TW + cc] = v.B[k];
    }
    Aff<NB> run;
    run.P = REV ? __shfl_down_sync(FULL, v.P, CW) : __shfl_up_sync(FULL, v.P, CW);
#pragma unroll
    for (int k = 0; k < NB; ++k) run.B[k] = REV ? __shfl_down_sync(FULL, v.B[k], CW) : __shfl_up_sync(FULL, v.B[k], CW);
    if (g == (REV ? GR - 1 : 0)) run = aff_identity<NB>();
    // exclusive prefixes of the group's segments
#pragma unroll
    for (int q = 0; q < MMAX; ++q) {
        const int sg = REV ? hi - 1 - q : lo + q;
        if (q < hi - lo) {
            Aff<NB> e;
            e.P = seg[(0 * S + sg) * (TW + 1) + cc];
#pragma unroll
            for (int k = 0; k < NB; ++k) e.B[k] = seg[((1 + k) * S + sg) * (TW + 1) + cc];
            seg[(0 * S + sg) * (TW + 1) + cc] = run.P;
#pragma unroll
            for (int k = 0; k < NB; ++k) seg[((1 + k) * S + sg) * (TW + 1) + cc] = run.B[k];
            run = aff_compose(run, e);
        }
    }
}

template <int NV>
constexpr int max_threads() { return NV == 1 ? 640 : (NV == 2 ? 448 : 352); }

// LSV: rows per warp segment; 16 for C_t >= 2 FILTER passes of images up to 16 x 320 rows
// (half the registers per thread, so 20 warps fit where 32-row segments allow 11-14)
// STRIPS: the tiles cover row strips of p.HS rows (tile -> (strip, column tile)); a separate
// instantiation so that the one-strip kernels keep their code
template <int CT, int MODE, bool PRE, int LSV = LS, bool STRIPS = false>
__global__ void __launch_bounds__(LSV == 12 ? 640 : LSV == 16 ? 640 : (LSV == 40 ? 512 : max_threads<(MODE == MODE_SUPPORT ? 1 : CT)>()), 1)
    k_col_cluster(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_d, const Params p) {
    constexpr int NV = (MODE == MODE_SUPPORT) ? 1 : CT;
    constexpr bool HASX = MODE != MODE_SUPPORT;
    // grouped segment scans (seg_scan_grp) in the one-channel throughput instantiations (row
    // strips, 40-row segments: many tile rounds per launch; C4 column pass 218-220 -> 214 us, the
    // step 32.10 -> 31.72 ms); one-round (latency-bound) images keep the per-column shuffle scans
    // (C1: 12.8 against 13.2 us), and so do the C_t = 3 instantiations, which are register-bound
    // (batched C3 with grouped scans: 460 against 432 us, the 12-row kernel spilling 16 B)
    constexpr bool GSCAN = (NV == 1 && (STRIPS || LSV == 40)) || LSV == 12;
    extern __shared__ __align__(128) float smem[];
    const int HB = p.HB, S = p.S, CB = p.CB;
    const Smem L = layout(NV, HB, S);
    float* lx = smem + L.land_x;
    float* ld = smem + L.land_d;
    float* segF = smem + L.segF;
    float* segR = smem + L.segR;
    float* totC = smem + L.totC;
    float* totA = smem + L.totA;
    float* remC = smem + L.remC;
    float* remA = smem + L.remA;
    float* carry = smem + L.carry;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* xbarC = bars + S;      // causal totals from the bands above have landed
    uint64_t* xbarA = bars + S + 1;  // anticausal totals from the bands below have landed

    const int c = threadIdx.x & 31;
    const int s = threadIdx.x >> 5;
    const int band = (int)cluster_ctarank();
    const int cluster = blockIdx.x / CB;
    const int nclusters = gridDim.x / CB;
    const int r0 = band * HB;
    const int lo = s * LSV;
    // PRE: d holds A1 = a_1^d and this pass's coefficient is A1^(2^nsq), nsq <= 3 (uniform)
    const int nsq = p.nsq;
    auto coef = [&](float v) {
        if constexpr (PRE) {
            float a1 = v;
            if (nsq > 0) a1 *= a1;
            if (nsq > 1) a1 *= a1;
            if (nsq > 2) a1 *= a1;
            return a1;
        } else {
            return coef_from_d(v, p.kc);
        }
    };

    const uint32_t xbytesC = (uint32_t)(band * (NV + 1) * TW * sizeof(float));
    const uint32_t xbytesA = (uint32_t)((CB - 1 - band) * (NV + 1) * TW * sizeof(float));
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
        mbar_init(xbarC, 1);
        mbar_init(xbarA, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(xbarC, xbytesC);  // armed for the first tile
        mbar_arrive_expect_tx(xbarA, xbytesA);
        tma_prefetch_desc(&tm_d);
        if (HASX) tma_prefetch_desc(&tm_x);
    }
    cluster_sync_all();  // every exchange barrier of the cluster is initialised and armed
    if (p.pdl_early) pdl_trigger();
    pdl_wait();  // the previous kernel's output (this pass's input X) is complete

    // lane 0 of warp q: TMA boxes of segment q of `tile` into the landing zone (every warp
    // issues its own segment's loads, so no warp carries the whole tile's issue)
    // tile -> (row strip, column tile): a strip of HS rows is filtered with zero carries at its
    // top and the link below it cut (the seam fix-up adds the carries)
    auto stage_seg = [&](int tile, int q) {
        const int col0 = (STRIPS ? tile % p.ntc : tile) * TW;
        const int sb = STRIPS ? (tile / p.ntc) * p.HS : 0;
        const uint32_t box = (uint32_t)(LSV * TW * sizeof(float));
        const int rq = r0 + q * LSV;
        const uint32_t bytes = rq < (STRIPS ? min(p.HS, p.H - sb) : p.H) ? box * (1 + (HASX ? NV : 0)) : 0u;
        mbar_arrive_expect_tx(&bars[q], bytes);
        if (bytes) {
            tma_load_2d(ld + q * LSV * TW, &tm_d, col0, sb + rq, &bars[q]);
            if constexpr (HASX) {
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    tma_load_3d(lx + (v * HB + q * LSV) * TW, &tm_x, col0, sb + rq, v, &bars[q]);
            }
        }
    };
    if (c == 0 && cluster < p.ntiles) stage_seg(cluster, s);

    int k = 0;
    for (int tile = cluster; tile < p.ntiles; tile += nclusters, ++k) {
        const int col0 = (STRIPS ? tile % p.ntc : tile) * TW;
        const int sb = STRIPS ? (tile / p.ntc) * p.HS : 0;  // first row of this tile's strip
        const int Hs = STRIPS ? min(p.HS, p.H - sb) : p.H;  // rows of the strip
        const int col = col0 + c;
        const bool colok = col < p.W;

        // ---- 1. landing zone -> registers; refill with the next tile ----
        // coefficient linking this segment's last row to the next row (the next segment's
        // first row, or the next band's): straight from global -- L2-resident, as the TMA
        // just brought it -- so no warp reads another warp's part of the landing zone
        float anext = 0.f;
        {
            const int rn = r0 + lo + LSV;
            if (colok && rn < Hs) anext = __ldg(p.d + (int64_t)(sb + rn) * p.pitch + col);
        }
        mbar_wait(&bars[s], (uint32_t)(k & 1));
        float a[LSV];
        float xv[NV][LSV];
        if (r0 + lo + LSV <= Hs) {
            // every row of the segment is in the image (warp-uniform): no per-row checks.
            // Lanes past W read the row padding; their values stay in their own column
            // (every step of the pass is per column) and are never stored.
            const float* ldc = ld + lo * TW + c;
#pragma unroll
            for (int j = 0; j < LSV; ++j) {
                a[j] = coef(ldc[j * TW]);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) xv[v][j] = lx[(v * HB + lo + j) * TW + c];
                    else xv[v][j] = 0.f;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < LSV; ++j) {
                const int rr = lo + j;
                const bool ok = colok && (r0 + rr) < Hs;
                a[j] = ok ? coef(ld[rr * TW + c]) : 0.f;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) xv[v][j] = ok ? lx[(v * HB + rr) * TW + c] : 0.f;
                    else xv[v][j] = 0.f;
                }
            }
        }
        // coefficient linking this segment's last row to the next row: from the
        // landing zone (next segment; it landed before the barrier below) or, for the
        // band's last segment, straight from global (first row of the next band)
        if (colok && r0 + lo + LSV < Hs) anext = coef(anext);
        // this warp's segment is in registers: refill it with the next tile (only this warp
        // reads it, so no CTA barrier; the next tile's shared-memory scratch writes are
        // ordered by the fold barrier below, which every warp passes after this tile)
        __syncwarp();
        if (c == 0 && tile + nclusters < p.ntiles) stage_seg(tile + nclusters, s);

        // ---- 2. causal fold, segment scan, band total ----
        // Pin = a[1] ... a[LSV-1] serves both maps: the causal product is a[0] Pin, the
        // anticausal one (the step at j uses a[j + 1]) Pin anext
        float Pin = 1.f;
        {
            Aff<NV> m = aff_identity<NV>();
#pragma unroll
            for (int j = 0; j < LSV; ++j) {
                if (j > 0) Pin *= a[j];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) m.B[v] = fmaf(a[j], m.B[v] - xv[v][j], xv[v][j]);
                    else m.B[v] = fmaf(a[j], m.B[v], 1.f);
                }
            }
            m.P = a[0] * Pin;
            segF[(0 * S + s) * (TW + 1) + c] = m.P;
#pragma unroll
            for (int v = 0; v < NV; ++v) segF[((1 + v) * S + s) * (TW + 1) + c] = m.B[v];
        }
        __syncthreads();
        if (GSCAN && S <= 24) {  // grouped scans: 8 warps of 4 columns
            for (int w8 = s; w8 < 8; w8 += S) seg_scan_grp<NV, false, 8>(segF, S, w8, totC);
        } else if (S <= 16) {  // two columns per warp (the 40-row instantiation has S = 16)
            for (int cc = s; cc < TW / 2; cc += S) seg_scan2<NV, false>(segF, S, cc, cc + TW / 2, totC);
        } else {
            for (int cc = s; cc < TW; cc += S) seg_scan<NV, false>(segF, S, cc, totC);
        }
        __syncthreads();

        // ---- 3. push this band's causal total to every band below it (st.async into their
        //         shared memory, completing on their exchange barrier); warp 0 waits for the
        //         totals of the bands above and composes the causal carry ----
        for (int q = band + 1 + s; q < CB; q += S) {
#pragma unroll
            for (int k2 = 0; k2 < NV + 1; ++k2)
                st_async_f32(remC + (band * (NV + 1) + k2) * TW + c, totC[k2 * TW + c], xbarC, (uint32_t)q);
        }
        if (s == 0) {
            mbar_wait_cluster(xbarC, (uint32_t)(k & 1));
            if (c == 0) mbar_arrive_expect_tx(xbarC, xbytesC);  // re-arm for the next tile
            float cin[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) cin[v] = 0.f;
            for (int q = 0; q < band; ++q) {
                const float P = remC[(q * (NV + 1)) * TW + c];
#pragma unroll
                for (int v = 0; v < NV; ++v) cin[v] = fmaf(P, cin[v], remC[(q * (NV + 1) + 1 + v) * TW + c]);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) carry[v * TW + c] = cin[v];
        }
        __syncthreads();
        {
            const float eP = segF[(0 * S + s) * (TW + 1) + c];
            float y[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) y[v] = fmaf(eP, carry[v * TW + c], segF[((1 + v) * S + s) * (TW + 1) + c]);
            float Q = 1.f, E[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) E[v] = 0.f;
            if constexpr (HASX) {
                // exact causal apply, then the anticausal map of the segment folded bottom-up
                // (E = a_{j+1} (E - y_j) + y_j: two instructions per row and channel)
#pragma unroll
                for (int j = 0; j < LSV; ++j) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        y[v] = fmaf(a[j], y[v] - xv[v][j], xv[v][j]);
                        xv[v][j] = y[v];
                    }
                }
#pragma unroll
                for (int j = LSV - 1; j >= 0; --j) {
                    const float an = (j + 1 < LSV) ? a[j + 1] : anext;
#pragma unroll
                    for (int v = 0; v < NV; ++v) E[v] = fmaf(an, E[v] - xv[v][j], xv[v][j]);
                }
                Q = Pin * anext;
            } else {
#pragma unroll
                for (int j = 0; j < LSV; ++j) {
                    const float an = (j + 1 < LSV) ? a[j + 1] : anext;
                    y[0] = fmaf(a[j], y[0], 1.f);
                    xv[0][j] = y[0];
                    E[0] += Q;
                    Q *= an;
                }
            }
            segR[(0 * S + s) * (TW + 1) + c] = Q;
#pragma unroll
            for (int v = 0; v < NV; ++v) segR[((1 + v) * S + s) * (TW + 1) + c] = E[v];
        }
        __syncthreads();
        if (GSCAN && S <= 24) {
            for (int w8 = s; w8 < 8; w8 += S) seg_scan_grp<NV, true, 8>(segR, S, w8, totA);
        } else if (S <= 16) {
            for (int cc = s; cc < TW / 2; cc += S) seg_scan2<NV, true>(segR, S, cc, cc + TW / 2, totA);
        } else {
            for (int cc = s; cc < TW; cc += S) seg_scan<NV, true>(segR, S, cc, totA);
        }
        __syncthreads();

        // ---- 4. anticausal totals flow upwards the same way ----
        for (int q = band - 1 - s; q >= 0; q -= S) {
#pragma unroll
            for (int k2 = 0; k2 < NV + 1; ++k2)
                st_async_f32(remA + (band * (NV + 1) + k2) * TW + c, totA[k2 * TW + c], xbarA, (uint32_t)q);
        }
        if (s == 0) {
            mbar_wait_cluster(xbarA, (uint32_t)(k & 1));
            if (c == 0) mbar_arrive_expect_tx(xbarA, xbytesA);
            float ein[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) ein[v] = 0.f;
            for (int q = CB - 1; q > band; --q) {
                const float Qb = remA[(q * (NV + 1)) * TW + c];
#pragma unroll
                for (int v = 0; v < NV; ++v) ein[v] = fmaf(Qb, ein[v], remA[(q * (NV + 1) + 1 + v) * TW + c]);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) carry[v * TW + c] = ein[v];
        }
        __syncthreads();
        {
            const float eQ = segR[(0 * S + s) * (TW + 1) + c];
            float z[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) z[v] = fmaf(eQ, carry[v * TW + c], segR[((1 + v) * S + s) * (TW + 1) + c]);
#pragma unroll
            for (int j = LSV - 1; j >= 0; --j) {
                const float an = (j + 1 < LSV) ? a[j + 1] : anext;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float yv = xv[v][j];
                    if constexpr (HASX) {
                        z[v] = fmaf(an, z[v] - yv, yv);
                        xv[v][j] = z[v];
                    } else {
                        z[v] = fmaf(an, z[v], 1.f);
                        xv[v][j] = yv + z[v] - 1.f;  // s_y = P + Q - 1
                    }
                }
            }
        }

        // ---- 5. write-out straight from registers ----
        {
            const int nrow = min(LSV, Hs - (r0 + lo));
            if (colok && nrow > 0) {
                if constexpr (MODE == MODE_FILTER || MODE == MODE_SUPPORT) {
                    float* base = (MODE == MODE_FILTER ? p.x : p.support) + (int64_t)(sb + r0 + lo) * p.pitch + col;
                    const int64_t pitch = p.pitch;
                    if (nrow == LSV) {  // full segment: a running pointer, no per-row checks
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            float* q = base + v * p.plane;
#pragma unroll
                            for (int j = 0; j < LSV; ++j, q += pitch) *q = xv[v][j];
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < LSV; ++j)
                            if (j < nrow) {
#pragma unroll
                                for (int v = 0; v < NV; ++v) base[v * p.plane + (int64_t)j * pitch] = xv[v][j];
                            }
                    }
                }
            }
            // row strips: the strip's last and first output rows, for the seam fix-up (which must
            // read them before it corrects the rows around the seam)
            if constexpr (STRIPS) {  // seam strips of one image (batched contexts pass no sedge)
              if (p.sedge) {
                const int strip = tile / p.ntc;
                const int64_t ew = (int64_t)p.ntc * TW, ec = (int64_t)(tile % p.ntc) * TW + c;
                const int jl = Hs - 1 - (r0 + lo);
                if (jl >= 0 && jl < LSV) {  // warp-uniform
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        float yl = xv[v][0];
#pragma unroll
                        for (int j = 1; j < LSV; ++j) yl = (j == jl) ? xv[v][j] : yl;
                        p.sedge[((int64_t)(strip * 2 + 0) * NV + v) * ew + ec] = yl;
                    }
                }
                if (r0 + lo == 0) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) p.sedge[((int64_t)(strip * 2 + 1) * NV + v) * ew + ec] = xv[v][0];
                }
              }
            }
        }
        // no barrier here: before the next tile's fold barrier a warp writes only its own
        // segF slot and its own part of the landing zone, which no other warp reads after
        // the anticausal carry barrier of this tile
    }
    // the next kernel may launch once every CTA is here (triggering at the start lets its CTAs
    // take SM resources while this persistent grid runs)
    if (!p.pdl_early) pdl_trigger();
    cluster_sync_all();  // no CTA leaves while another may still read its shared memory
}


// ---------------------------------------------------------------------------------------
// Row-band variant.  A separate kernel so that the single-GPU
// instantiations above keep their exact code: MODE_TUPLE emits the rank band's 5-tuple
// (one extra channel, the carry sensitivity); BAND FILTER takes external carries and, for
// the edge fix-up scheme, exports y at row H - 1 and z at row 0.
struct BandParams : Params {
    // APPLY carries into the rank band (causal c at the top, anticausal e at the bottom),
    // [ntiles][2][CT][TW]; TUPLE output [ntiles][2CT+3][TW]; edge scheme [ntiles][2CT+1][TW]
    const float* ext;
    float* rank_tuples;
    float* edge;
};

// NX planes of x staged per tile, NV channels carried (TUPLE: NX + 1)
__host__ __device__ inline Smem layout_band(int NX, int NV, int HB, int S) {
    Smem L = layout(NV, HB, S);
    const int shrink = (NV - NX) * HB * TW;  // the carried-only channels are not staged
    L.land_d -= shrink;
    L.segF -= shrink;
    L.segR -= shrink;
    L.totC -= shrink;
    L.totA -= shrink;
    L.remC -= shrink;
    L.remA -= shrink;
    L.carry -= shrink;
    L.bars -= shrink;
    L.bytes -= (size_t)shrink * sizeof(float);
    return L;
}

template <int CT, int MODE>
__host__ __device__ constexpr int nchan() { return MODE == MODE_SUPPORT ? 1 : (MODE == MODE_TUPLE ? CT + 1 : CT); }

// BAND (row-band mode, MODE_TUPLE or FILTER with external carries): rows past H are identity
// maps and row H is the link to the next rank; the single-GPU instantiations keep the
// plain code (a = 0 past H, no external carries)
template <int CT, int MODE, bool PRE, bool BAND>
__global__ void __launch_bounds__(max_threads<nchan<CT, MODE>()>(), 1)
    k_col_cluster_band(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_d, const BandParams p) {
    // TUPLE: channel CT is the carry sensitivity g (x = 0, carry-in 1 at the rank band's top)
    constexpr int NV = nchan<CT, MODE>();
    constexpr int NX = (MODE == MODE_SUPPORT) ? 0 : CT;  // x planes staged
    constexpr bool HASX = MODE != MODE_SUPPORT;
    extern __shared__ __align__(128) float smem[];
    const int HB = p.HB, S = p.S, CB = p.CB;
    const Smem L = layout_band(NX, NV, HB, S);
    float* lx = smem + L.land_x;
    float* ld = smem + L.land_d;
    float* segF = smem + L.segF;
    float* segR = smem + L.segR;
    float* totC = smem + L.totC;
    float* totA = smem + L.totA;
    float* remC = smem + L.remC;
    float* remA = smem + L.remA;
    float* carry = smem + L.carry;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* xbarC = bars + S;      // causal totals from the bands above have landed
    uint64_t* xbarA = bars + S + 1;  // anticausal totals from the bands below have landed

    const int c = threadIdx.x & 31;
    const int s = threadIdx.x >> 5;
    const int band = (int)cluster_ctarank();
    const int cluster = blockIdx.x / CB;
    const int nclusters = gridDim.x / CB;
    const int r0 = band * HB;
    const int lo = s * LS;
    // PRE: d holds A1 = a_1^d and this pass's coefficient is A1^(2^nsq), nsq <= 3 (uniform)
    const int nsq = p.nsq;
    auto coef = [&](float v) {
        if constexpr (PRE) {
            float a1 = v;
            if (nsq > 0) a1 *= a1;
            if (nsq > 1) a1 *= a1;
            if (nsq > 2) a1 *= a1;
            return a1;
        } else {
            return coef_from_d(v, p.kc);
        }
    };

    const uint32_t xbytesC = (uint32_t)(band * (NV + 1) * TW * sizeof(float));
    const uint32_t xbytesA = (uint32_t)((CB - 1 - band) * (NV + 1) * TW * sizeof(float));
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
        mbar_init(xbarC, 1);
        mbar_init(xbarA, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(xbarC, xbytesC);  // armed for the first tile
        mbar_arrive_expect_tx(xbarA, xbytesA);
        tma_prefetch_desc(&tm_d);
        if (HASX) tma_prefetch_desc(&tm_x);
    }
    cluster_sync_all();  // every exchange barrier of the cluster is initialised and armed
    if (p.pdl_early) pdl_trigger();
    pdl_wait();

    auto stage_seg = [&](int tile, int q) {  // lane 0 of warp q: segment q of `tile`
        const int col0 = tile * TW;
        const uint32_t box = (uint32_t)(LS * TW * sizeof(float));
        const int rq = r0 + q * LS;
        const uint32_t bytes = rq < p.H ? box * (1 + NX) : 0u;
        mbar_arrive_expect_tx(&bars[q], bytes);
        if (bytes) {
            tma_load_2d(ld + q * LS * TW, &tm_d, col0, rq, &bars[q]);
#pragma unroll
            for (int v = 0; v < NX; ++v) tma_load_3d(lx + (v * HB + q * LS) * TW, &tm_x, col0, rq, v, &bars[q]);
        }
    };
    if (c == 0 && cluster < p.ntiles) stage_seg(cluster, s);

    int k = 0;
    for (int tile = cluster; tile < p.ntiles; tile += nclusters, ++k) {
        const int col0 = tile * TW;
        const int col = col0 + c;
        const bool colok = col < p.W;

        // external carries of this tile (APPLY), loaded now so their latency hides behind the fold
        float cx0[NV], ex0[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            cx0[v] = (MODE != MODE_TUPLE && s == 0 && p.ext) ? __ldg(p.ext + ((int64_t)tile * 2 * NV + v) * TW + c) : 0.f;
            ex0[v] = (MODE != MODE_TUPLE && s == 0 && p.ext) ? __ldg(p.ext + ((int64_t)tile * 2 * NV + NV + v) * TW + c)
                                                            : 0.f;
        }
        // ---- 1. landing zone -> registers; refill with the next tile ----
        // link coefficient of the segment's last row, raw from global (see the single-GPU
        // kernel): the next segment's first row, the next band's, or row H (the link below
        // the rank band); identity past it
        float anext = 0.f;
        {
            const int rn = r0 + lo + LS;
            const bool ld_ok = BAND ? (colok && rn <= p.H) : (colok && rn < p.H);
            if (ld_ok) anext = __ldg(p.d + (int64_t)rn * p.pitch + col);
        }
        mbar_wait(&bars[s], (uint32_t)(k & 1));
        float a[LS];
        float xv[NV][LS];
        if (r0 + lo + LS <= p.H) {
            // every row of the segment is in the image (warp-uniform): no per-row checks.
            // Lanes past W read the row padding; their values stay in their own column
            // (every step of the pass is per column) and are never stored.
            const float* ldc = ld + lo * TW + c;
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                a[j] = coef(ldc[j * TW]);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) xv[v][j] = v < NX ? lx[(v * HB + lo + j) * TW + c] : 0.f;
                    else xv[v][j] = 0.f;
                }
            }
        } else {
            // rows past H: row H carries the link coefficient to the rows below (d row H: the
            // next rank's first row in row-band mode, +inf -> 0 at the image bottom); the rows
            // after it are identity maps (a = 1, x = 0), so the causal map of the band stops at
            // row H - 1 and the anticausal carry from below reaches row H unchanged
            const float aH = (BAND && colok && r0 + lo <= p.H && p.H < r0 + lo + LS)
                                 ? coef(__ldg(p.d + (int64_t)p.H * p.pitch + col)) : 0.f;
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                const int rr = lo + j;
                const bool ok = colok && (r0 + rr) < p.H;
                if constexpr (BAND) a[j] = ok ? coef(ld[rr * TW + c]) : (!colok ? 0.f : (r0 + rr == p.H ? aH : 1.f));
                else a[j] = ok ? coef(ld[rr * TW + c]) : 0.f;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) xv[v][j] = (ok && v < NX) ? lx[(v * HB + rr) * TW + c] : 0.f;
                    else xv[v][j] = 0.f;
                }
            }
        }
        // coefficient linking this segment's last row to the next row: from the
        // landing zone (next segment; it landed before the barrier below) or, for the
        // band's last segment, straight from global (first row of the next band)
        // (row H of d is the link below the band: the next rank's first row in row-band mode,
        // +inf -- a = 0 -- at the image bottom)
        {
            const int rn = r0 + lo + LS;
            if constexpr (BAND) {
                if (colok) anext = rn > p.H ? 1.f : coef(anext);  // identity rows past the link
            } else {
                if (colok && rn < p.H) anext = coef(anext);
            }
        }
        __syncwarp();  // this warp's segment is in registers: refill it (only this warp reads it)
        if (c == 0 && tile + nclusters < p.ntiles) stage_seg(tile + nclusters, s);

        // ---- 2. causal fold, segment scan, band total ----
        {
            Aff<NV> m = aff_identity<NV>();
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                m.P *= a[j];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if constexpr (HASX) m.B[v] = fmaf(a[j], m.B[v] - xv[v][j], xv[v][j]);
                    else m.B[v] = fmaf(a[j], m.B[v], 1.f);
                }
            }
            segF[(0 * S + s) * (TW + 1) + c] = m.P;
#pragma unroll
            for (int v = 0; v < NV; ++v) segF[((1 + v) * S + s) * (TW + 1) + c] = m.B[v];
        }
        __syncthreads();
        for (int cc = s; cc < TW; cc += S) seg_scan<NV, false>(segF, S, cc, totC);
        __syncthreads();

        // ---- 3. push this band's causal total to every band below it (st.async into their
        //         shared memory, completing on their exchange barrier); warp 0 waits for the
        //         totals of the bands above and composes the causal carry ----
        for (int q = band + 1 + s; q < CB; q += S) {
#pragma unroll
            for (int k2 = 0; k2 < NV + 1; ++k2)
                st_async_f32(remC + (band * (NV + 1) + k2) * TW + c, totC[k2 * TW + c], xbarC, (uint32_t)q);
        }
        if (s == 0) {
            mbar_wait_cluster(xbarC, (uint32_t)(k & 1));
            if (c == 0) mbar_arrive_expect_tx(xbarC, xbytesC);  // re-arm for the next tile
            float cin[NV];  // carry into the rank band's top: 0, the APPLY carry, or 1 for g (TUPLE)
#pragma unroll
            for (int v = 0; v < NV; ++v)
                cin[v] = (MODE == MODE_TUPLE) ? (v == CT ? 1.f : 0.f) : cx0[v];
            for (int q = 0; q < band; ++q) {
                const float P = remC[(q * (NV + 1)) * TW + c];
#pragma unroll
                for (int v = 0; v < NV; ++v) cin[v] = fmaf(P, cin[v], remC[(q * (NV + 1) + 1 + v) * TW + c]);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) carry[v * TW + c] = cin[v];
        }
        __syncthreads();
        {
            const float eP = segF[(0 * S + s) * (TW + 1) + c];
            float y[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) y[v] = fmaf(eP, carry[v * TW + c], segF[((1 + v) * S + s) * (TW + 1) + c]);
            float Q = 1.f, E[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) E[v] = 0.f;
#pragma unroll
            for (int j = 0; j < LS; ++j) {
                const float an = (j + 1 < LS) ? a[j + 1] : anext;
                if constexpr (HASX) {
                    const float qb = Q * (1.f - an);
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        y[v] = fmaf(a[j], y[v] - xv[v][j], xv[v][j]);
                        xv[v][j] = y[v];
                        E[v] = fmaf(qb, y[v], E[v]);
                    }
                } else {
                    y[0] = fmaf(a[j], y[0], 1.f);
                    xv[0][j] = y[0];
                    E[0] += Q;
                }
                Q *= an;
            }
            segR[(0 * S + s) * (TW + 1) + c] = Q;
#pragma unroll
            for (int v = 0; v < NV; ++v) segR[((1 + v) * S + s) * (TW + 1) + c] = E[v];
}
        __syncthreads();
        for (int cc = s; cc < TW; cc += S) seg_scan<NV, true>(segR, S, cc, totA);
        __syncthreads();

        // ---- 4. anticausal totals flow upwards the same way ----
        for (int q = band - 1 - s; q >= 0; q -= S) {
#pragma unroll
            for (int k2 = 0; k2 < NV + 1; ++k2)
                st_async_f32(remA + (band * (NV + 1) + k2) * TW + c, totA[k2 * TW + c], xbarA, (uint32_t)q);
        }
        {  // row-band outputs at row H - 1, off the critical path: while the exchange runs
            // (its warp only, warp-uniform; xv still holds y): y of the x channels
            // (c = 0) and, in TUPLE mode, of g (c = 1) -- the rank band's causal map c_out = A c + B
            const int jl = p.H - 1 - (r0 + lo);
            if ((MODE == MODE_TUPLE || p.edge) && jl >= 0 && jl < LS) {
                float yl[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    yl[v] = xv[v][0];
#pragma unroll
                    for (int j = 1; j < LS; ++j) yl[v] = (j == jl) ? xv[v][j] : yl[v];
                }
                if (colok) {
                    if constexpr (MODE == MODE_TUPLE) {
                        float* rt = p.rank_tuples + (int64_t)tile * (2 * CT + 3) * TW;
                        rt[0 * TW + c] = yl[CT];
#pragma unroll
                        for (int v = 0; v < CT; ++v) rt[(1 + v) * TW + c] = yl[v];
                    } else {
                        float* ed = p.edge + (int64_t)tile * (2 * CT + 1) * TW;
#pragma unroll
                        for (int v = 0; v < CT; ++v) ed[v * TW + c] = yl[v];
                    }
                }
            }
        }
        if (s == 0) {
            mbar_wait_cluster(xbarA, (uint32_t)(k & 1));
            if (c == 0) mbar_arrive_expect_tx(xbarA, xbytesA);
            float ein[NV];  // carry into the rank band's bottom: 0 or the APPLY carry
#pragma unroll
            for (int v = 0; v < NV; ++v)
                ein[v] = (MODE != MODE_TUPLE) ? ex0[v] : 0.f;
            float Qbe = 1.f;
            for (int q = CB - 1; q > band; --q) {
                const float Qb = remA[(q * (NV + 1)) * TW + c];
                if constexpr (MODE == MODE_TUPLE) Qbe *= Qb;
#pragma unroll
                for (int v = 0; v < NV; ++v) ein[v] = fmaf(Qb, ein[v], remA[(q * (NV + 1) + 1 + v) * TW + c]);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) carry[v * TW + c] = ein[v];
            if (MODE == MODE_TUPLE && band == 0) {  // rank anticausal map: e_top = Z0 + S c + Q e
                float* rt = p.rank_tuples + (int64_t)tile * (2 * CT + 3) * TW;
                const float Qown = totA[0 * TW + c];
                rt[(1 + CT) * TW + c] = Qbe * Qown;
#pragma unroll
                for (int v = 0; v < CT; ++v) rt[(2 + CT + v) * TW + c] = fmaf(Qown, ein[v], totA[(1 + v) * TW + c]);
                rt[(2 + 2 * CT) * TW + c] = fmaf(Qown, ein[CT], totA[(1 + CT) * TW + c]);
            }
        }
        __syncthreads();
        if constexpr (MODE != MODE_TUPLE) {
            const float eQ = segR[(0 * S + s) * (TW + 1) + c];
            float z[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) z[v] = fmaf(eQ, carry[v * TW + c], segR[((1 + v) * S + s) * (TW + 1) + c]);
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
                        z[v] = fmaf(an, z[v], 1.f);
                        xv[v][j] = yv + z[v] - 1.f;  // s_y = P + Q - 1
                    }
                }
            }
        }

        if constexpr (BAND && MODE == MODE_FILTER) {  // edge scheme: z at row 0 (c = e = 0)
            if (p.edge && colok && band == 0 && s == 0) {
                float* ed = p.edge + (int64_t)tile * (2 * CT + 1) * TW;
#pragma unroll
                for (int v = 0; v < CT; ++v) ed[(CT + v) * TW + c] = xv[v][0];
            }
        }
        // ---- 5. write-out straight from registers (TUPLE: nothing; the tuple is written) ----
        if constexpr (MODE != MODE_TUPLE) {
            const int nrow = min(LS, p.H - (r0 + lo));
            if (colok && nrow > 0) {
                if constexpr (MODE == MODE_FILTER || MODE == MODE_SUPPORT) {
                    float* base = (MODE == MODE_FILTER ? p.x : p.support) + (int64_t)(r0 + lo) * p.pitch + col;
                    const int64_t pitch = p.pitch;
                    if (nrow == LS) {  // full segment: a running pointer, no per-row checks
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            float* q = base + v * p.plane;
#pragma unroll
                            for (int j = 0; j < LS; ++j, q += pitch) *q = xv[v][j];
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < LS; ++j)
                            if (j < nrow) {
#pragma unroll
                                for (int v = 0; v < NV; ++v) base[v * p.plane + (int64_t)j * pitch] = xv[v][j];
                            }
                    }
                }
            }
        }
        // no barrier here: before the next tile's fold barrier a warp writes only its own
        // segF slot and its own part of the landing zone (as in the single-GPU kernel)
    }
    // the next kernel may launch once every CTA is here (triggering at the start lets its CTAs
    // take SM resources while this persistent grid runs)
    if (!p.pdl_early) pdl_trigger();
    cluster_sync_all();  // no CTA leaves while another may still read its shared memory
}

}  // namespace colc

// ---------------------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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

// Tensor maps are pure functions of their encode arguments; the column passes of a solve reuse
// the same few (X and the coefficient plane), so they are encoded once and cached (the encode
// is host work on every eager launch otherwise).
struct TmapKey {
    const void* base;
    int64_t pitch, H, planes;
    int rank, box_rows;
    bool operator==(const TmapKey& o) const {
        return base == o.base && pitch == o.pitch && H == o.H && planes == o.planes && rank == o.rank &&
               box_rows == o.box_rows;
    }
};

static bool tmap_encode(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int64_t planes, int rank,
                        int box_rows);

static bool tmap(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int64_t planes, int rank,
                 int box_rows = colc::LS) {
    static std::mutex mu;
    static std::vector<std::pair<TmapKey, CUtensorMap>> cache;  // most recent last, <= 64 entries
    const TmapKey key{base, pitch, H, planes, rank, box_rows};
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = cache.rbegin(); it != cache.rend(); ++it)
            if (it->first == key) {
                *m = it->second;
                return true;
            }
    }
    if (!tmap_encode(m, base, pitch, H, planes, rank, box_rows)) return false;
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 64) cache.erase(cache.begin());
    cache.emplace_back(key, *m);
    return true;
}

static bool tmap_encode(CUtensorMap* m, const void* base, int64_t pitch, int64_t H, int64_t planes, int rank,
                        int box_rows) {
    auto enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)H, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * sizeof(float)), (cuuint64_t)(pitch * H * sizeof(float))};
    cuuint32_t box[3] = {(cuuint32_t)colc::TW, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CT, int MODE, bool PRE = false>
static const void* kptr() {
    return reinterpret_cast<const void*>(colc::k_col_cluster<CT, MODE, PRE>);
}
template <int CT, int MODE, bool PRE = false>
static const void* kptr_band() {
    return reinterpret_cast<const void*>(colc::k_col_cluster_band<CT, MODE, PRE, true>);
}
template <int CT, bool PRE, int LSV = 16>
static const void* kptr16() {
    return reinterpret_cast<const void*>(colc::k_col_cluster<CT, MODE_FILTER, PRE, LSV>);
}
static const void* colc_kernel(int Ct, int mode, bool pre = false, bool band = false, int ls = colc::LS,
                               bool strips = false) {
    if (strips) {  // row strips: FILTER on the pass-1 coefficient (plan_strips, batched contexts)
        if (mode != MODE_FILTER || band || !pre) return nullptr;
        if (Ct == 1 && ls == 40) return reinterpret_cast<const void*>(colc::k_col_cluster<1, MODE_FILTER, true, 40, true>);
        if (Ct == 1 && ls == 32) return reinterpret_cast<const void*>(colc::k_col_cluster<1, MODE_FILTER, true, 32, true>);
        if (Ct == 2 && ls == 16) return reinterpret_cast<const void*>(colc::k_col_cluster<2, MODE_FILTER, true, 16, true>);
        if (Ct == 3 && ls == 16) return reinterpret_cast<const void*>(colc::k_col_cluster<3, MODE_FILTER, true, 16, true>);
        if (Ct == 3 && ls == 12) return reinterpret_cast<const void*>(colc::k_col_cluster<3, MODE_FILTER, true, 12, true>);
        return nullptr;
    }
    if (ls == 12) {  // C_t = 3 FILTER: 12-row segments, up to 24 warps per CTA
        if (mode != MODE_FILTER || band || Ct != 3) return nullptr;
        return pre ? kptr16<3, true, 12>() : kptr16<3, false, 12>();
    }
    if (ls == 40) {  // 16 warps x 40-row segments, C_t = 1 FILTER
        if (mode != MODE_FILTER || band || Ct != 1) return nullptr;
        return pre ? reinterpret_cast<const void*>(colc::k_col_cluster<1, MODE_FILTER, true, 40>)
                   : reinterpret_cast<const void*>(colc::k_col_cluster<1, MODE_FILTER, false, 40>);
    }
    if (ls == 16) {  // FILTER, C_t >= 2, single context
        if (mode != MODE_FILTER || band) return nullptr;
        switch (Ct * 2 + (pre ? 1 : 0)) {
            case 4: return kptr16<2, false>();
            case 5: return kptr16<2, true>();
            case 6: return kptr16<3, false>();
            case 7: return kptr16<3, true>();
        }
        return nullptr;
    }
    if (mode == MODE_SUPPORT) return kptr<1, MODE_SUPPORT>();
    if (band && mode == MODE_FILTER) {  // APPLY of the row-band exchange / the edge scheme's pass
        switch (Ct * 2 + (pre ? 1 : 0)) {
            case 2: return kptr_band<1, MODE_FILTER>();
            case 3: return kptr_band<1, MODE_FILTER, true>();
            case 4: return kptr_band<2, MODE_FILTER>();
            case 5: return kptr_band<2, MODE_FILTER, true>();
            case 6: return kptr_band<3, MODE_FILTER>();
            case 7: return kptr_band<3, MODE_FILTER, true>();
        }
        return nullptr;
    }
    if (pre && mode == MODE_FILTER) {
        switch (Ct) {
            case 1: return kptr<1, MODE_FILTER, true>();
            case 2: return kptr<2, MODE_FILTER, true>();
            case 3: return kptr<3, MODE_FILTER, true>();
        }
        return nullptr;
    }
    if (mode == MODE_TUPLE) {
        switch (Ct) {
            case 1: return kptr_band<1, MODE_TUPLE>();
            case 2: return kptr_band<2, MODE_TUPLE>();
            case 3: return kptr_band<3, MODE_TUPLE>();
        }
        return nullptr;
    }
    switch (Ct * 4 + mode) {
        case 4 + MODE_FILTER: return kptr<1, MODE_FILTER>();
        case 8 + MODE_FILTER: return kptr<2, MODE_FILTER>();
        case 12 + MODE_FILTER: return kptr<3, MODE_FILTER>();
    }
    return nullptr;
}

bool colc_strips_supported(int Ct, int ls) { return colc_kernel(Ct, MODE_FILTER, true, false, ls, true) != nullptr; }

// Fast path if the column fits a cluster of <= 16 CTAs with register-resident segments.
// ls: rows per warp segment, 32 (every mode) or 16 (FILTER at C_t >= 2, single context).
// Cluster size CB: its CTAs hold H / CB rows in <= 20 warps.  32-row segments: the smallest
// such CB (fewest exchange participants; one-round images are latency-bound: C1 at CB 2,
// 16 warps 14.4 us, at CB 9, 4 warps 20.8 us).  16-row segments: the fewest tile rounds
// (ceil(tiles / resident clusters); residency depends on how CB packs into the GPCs), ties
// to the larger CB (fewer warps per CTA): C3 CB 7 / 8 / 9 all give 15 clusters and 8 rounds,
// 84 / 80 / 78 us; CB 10 11 clusters, 101 us; CB 14 9 rounds, 97 us.  Plans are cached per
// device and shape (the occupancy queries cost host time on every solve).
static cudaError_t plan_col_cluster_uncached(const Geometry& g, int Ct, int mode, ColPlan* plan, int ls, int fcb) {
    const int NV = (mode == MODE_SUPPORT) ? 1 : (mode == MODE_TUPLE ? Ct + 1 : Ct);
    const int NX = (mode == MODE_SUPPORT) ? 0 : Ct;
    const void* fn = colc_kernel(Ct, mode, false, false, ls);
    if (!fn) return cudaErrorNotSupported;
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return e;
    int Smax = fa.maxThreadsPerBlock / colc::TW;
    if (Smax > (ls >= 16 ? 20 : 24)) Smax = ls >= 16 ? 20 : 24;
    // attributes are per function and shared by every plan: allow non-portable clusters and
    // the opt-in shared memory maximum (so that no plan lowers another's limit); the
    // A1-input (and, at 32-row segments, row-band) variants of the FILTER kernel get the same
    int optin = 0, dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
        return e;
    const bool f32 = mode == MODE_FILTER && ls == colc::LS;
    const bool strip = mode == MODE_FILTER && ((Ct == 1 && (ls == 32 || ls == 40)) || (Ct >= 2 && ls <= 16));
    for (const void* f : {fn, mode == MODE_FILTER ? colc_kernel(Ct, mode, true, false, ls) : fn,
                          f32 ? colc_kernel(Ct, mode, false, true) : fn, f32 ? colc_kernel(Ct, mode, true, true) : fn,
                          strip ? colc_kernel(Ct, mode, true, false, ls, true) : fn}) {
        if (!f) continue;
        cudaFuncAttributes fa2;
        if ((e = cudaFuncGetAttributes(&fa2, f)) != cudaSuccess) return e;
        if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - (int)fa2.sharedSizeBytes)) != cudaSuccess)
            return e;
    }
    const int ntiles = (int)((g.W + colc::TW - 1) / colc::TW);
    int64_t best_cost = -1;
    for (int CB = fcb ? fcb : 1; CB <= (fcb ? fcb : 16); ++CB) {
        const int64_t HBmin = (g.H + CB - 1) / CB;
        const int S = (int)((HBmin + ls - 1) / ls);
        if (S > Smax) continue;
        const int HB = S * ls;
        const colc::Smem L = mode == MODE_TUPLE ? colc::layout_band(NX, NV, HB, S) : colc::layout(NV, HB, S);
        if (L.bytes > 227 * 1024) continue;
        // how many clusters can be resident at once
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)CB, 1, 1);
        cfg.blockDim = dim3((unsigned)(colc::TW * S), 1, 1);
        cfg.dynamicSmemBytes = L.bytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)CB;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
        if (e != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            continue;
        }
        if (nclusters > ntiles) nclusters = ntiles;
        const int64_t cost = (ntiles + nclusters - 1) / nclusters;  // tile rounds
        if (best_cost >= 0 && (ls == colc::LS || cost > best_cost)) continue;
        best_cost = cost;
        plan->kind = 1;
        plan->TW = colc::TW;
        plan->CB = CB;
        plan->HB = HB;
        plan->S = S;
        plan->Ls = ls;
        plan->nb = CB;
        plan->ntiles = ntiles;
        plan->threads = colc::TW * S;
        plan->grid = dim3((unsigned)(CB * nclusters), 1, 1);
        plan->smem = L.bytes;
        plan->tuple_floats = 0;
        plan->flag_count = 0;
        if (ls == colc::LS) break;
    }
    return best_cost >= 0 ? cudaSuccess : cudaErrorNotSupported;
}

cudaError_t plan_col_cluster_ls(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan, int ls, int force_cb) {
    (void)num_sms;
    const int fcb = force_cb >= 0 ? force_cb : option_col_cluster();  // forced cluster size (0 = auto)
    int dev = 0;
    cudaGetDevice(&dev);
    struct Entry {
        int dev, Ct, mode, ls, fcb;
        int64_t H, W;
        cudaError_t err;
        ColPlan plan;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Entry& en : cache)
            if (en.dev == dev && en.Ct == Ct && en.mode == mode && en.ls == ls && en.fcb == fcb && en.H == g.H &&
                en.W == g.W) {
                if (en.err == cudaSuccess) *plan = en.plan;
                return en.err;
            }
    }
    ColPlan p{};
    const cudaError_t e = plan_col_cluster_uncached(g, Ct, mode, &p, ls, fcb);
    if (e != cudaSuccess) cudaGetLastError();
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() < 256) cache.push_back(Entry{dev, Ct, mode, ls, fcb, g.H, g.W, e, p});
    if (e == cudaSuccess) *plan = p;
    return e;
}

cudaError_t plan_col_cluster(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan) {
    return plan_col_cluster_ls(g, Ct, mode, num_sms, plan, colc::LS);
}

cudaError_t launch_col_cluster(const ColPlan& plan, const Geometry& g, int Ct, int mode, float* x, const float* d,
                               float kc, const UpdateArgs* upd, float* support, cudaStream_t s, int nsq,
                               const float* ext, float* rank_tuples, float* edge, float* sedge, float* x_out) {
    colc::BandParams p = {};
    p.sedge = sedge;
    p.nsq = nsq;
    p.ext = ext;
    p.rank_tuples = rank_tuples;
    p.edge = edge;
    p.x = x_out ? x_out : x;  // the TMA reads x; the stores go to p.x
    p.d = d;
    p.support = support;
    if (upd) p.upd = *upd;
    p.plane = g.plane;
    p.pitch = g.pitch;
    p.H = (int)g.H;
    p.W = (int)g.W;
    p.HB = plan.HB;
    p.S = plan.S;
    p.CB = plan.CB;
    p.ntiles = plan.ntiles;
    p.HS = plan.HS > 0 ? plan.HS : (int)g.H;
    p.ntc = plan.ntc > 0 ? plan.ntc : plan.ntiles;
    p.kc = kc;
    // PDL trigger at the end of the kernel (option pdl = 2: at the start, for experiments; a
    // start trigger was never faster, and 20-30% slower on mid-size images)
    p.pdl_early = option_pdl() == 2;
    CUtensorMap tx, td;
    if (!tmap(&td, d, g.pitch, g.H, 1, 2, plan.Ls)) return cudaErrorInvalidValue;
    if (mode != MODE_SUPPORT) {
        if (!tmap(&tx, x, g.pitch, g.H, Ct, 3, plan.Ls)) return cudaErrorInvalidValue;
    } else {
        tx = td;
    }
    const void* fn = colc_kernel(Ct, mode, nsq >= 0, ext != nullptr || edge != nullptr, plan.Ls, plan.HS > 0);
    if (!fn) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = plan.grid;
    cfg.blockDim = dim3((unsigned)plan.threads, 1, 1);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)plan.CB;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (dts_device.cuh)
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // PDL only when the grid has at most one CTA per SM: a grid of several CTAs per SM launched
    // early lands its clusters on the SMs the previous kernel frees first, several to an SM,
    // and keeps that imbalance for the whole persistent launch (7071 x 10000, 4 row strips of
    // 405 CTAs: 27 ms per solve with PDL, 22.5 without)
    static std::atomic<int> nsm_dev[64];  // SM count per device (0: not queried yet)
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64) {
        nsm = nsm_dev[dev].load(std::memory_order_relaxed);
        if (nsm < 1) {
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            if (nsm < 1) nsm = 1;
            nsm_dev[dev].store(nsm, std::memory_order_relaxed);
        }
    }
    cfg.numAttrs = (option_pdl() && plan.grid.x <= (unsigned)nsm) ? 2 : 1;
    void* args[] = {&tx, &td, &p};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Row-band edge fix-up scheme.  A carry entering a band at its top
// edge changes y by c G_k (G_k = prod_{j<=k} a_j) and z by c Gamma_k (Gamma = the anticausal
// response of G); one entering at the bottom changes z by e Theta_k (Theta_k =
// prod_{j=k+1..H} a_j).  Both decay at least like a_i^k; past L rows they are below fp32
// resolution, so with bands of >= 2L rows the banded pass is the zero-carry pass plus
// these two corrections on the L rows at each edge.

// per column, sequential over the edge rows (create time): Gamma (top L rows), Theta
// (bottom L rows, row H - L first); d has rows 0..H (row H: the link below the band)
__global__ void k_edge_profiles(const float* __restrict__ d, int64_t H, int64_t W, int64_t pitch, int L, float kc,
                                float* __restrict__ gam, float* __restrict__ theta, bool raw) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= W) return;
    float G = 1.f;
#pragma unroll 8
    for (int k = 0; k < L; ++k) {  // G_k = prod_{j <= k} a_j (a_0: the link to the band above)
        G *= coef_from_d(__ldg(d + (int64_t)k * pitch + col), kc);
        gam[(int64_t)k * pitch + col] = G;
    }
    float dz = 0.f;  // anticausal response, zero at row L (below resolution); raw: keep G itself
#pragma unroll 8
    for (int k = L - 1; k >= 0 && !raw; --k) {
        const float an = coef_from_d(__ldg(d + (int64_t)(k + 1) * pitch + col), kc);
        const float g = gam[(int64_t)k * pitch + col];
        dz = fmaf(an, dz - g, g);
        gam[(int64_t)k * pitch + col] = dz;
    }
    float th = coef_from_d(__ldg(d + H * pitch + col), kc);  // a_H
#pragma unroll 8
    for (int64_t k = H - 1; k >= H - L; --k) {
        theta[(k - (H - L)) * pitch + col] = th;
        th *= coef_from_d(__ldg(d + k * pitch + col), kc);
    }
}

cudaError_t launch_edge_profiles(const float* d, const Geometry& g, int L, float kc, float* gam, float* theta,
                                 cudaStream_t s, bool raw) {
    k_edge_profiles<<<(unsigned)((g.W + 127) / 128), 128, 0, s>>>(d, g.H, g.W, g.pitch, L, kc, gam, theta, raw);
    return cudaGetLastError();
}

// Row-strip seam fix-up (single-GPU tall images).  Strip j starts at row
// j HS; the FILTER pass ran every strip with a zero carry at its top and the link below it cut.
// With y_last (strip j - 1's last output row) and z0 (strip j's first), both uncorrected, the
// fix-up adds c Gamma_j on strip j's top L rows and e Theta_{j-1} on strip j - 1's bottom L rows,
// c = y_last, e = z0 + y_last Gamma_j[0] - y_last (reading R26: the algebra of the row-band edge
// scheme, on one GPU).  Seams touch disjoint rows (2L < HS).
// The edge values come from the column kernel (sedge), so every corrected row is independent:
// thread = (column, seam, 8 consecutive rows of the 2L-row window around the seam).
__global__ void __launch_bounds__(128) k_seam_fix(float* __restrict__ x, int Ct, int64_t W, int64_t pitch,
                                                  int64_t plane, int HS, int L, int ntc,
                                                  const float* __restrict__ gam, const float* __restrict__ theta,
                                                  const float* __restrict__ sedge) {
    const int64_t col = (int64_t)blockIdx.x * 128 + threadIdx.x;
    const int j = blockIdx.y + 1;  // seam between strips j - 1 and j
    const int k0 = blockIdx.z * 8;
    pdl_wait();
    if (col >= W) return;
    const int64_t s0 = (int64_t)j * HS, ew = (int64_t)ntc * 32;
    const float g0 = __ldg(gam + (int64_t)j * L * pitch + col);
    for (int v = 0; v < Ct; ++v) {
        const float yl = __ldg(sedge + ((int64_t)((j - 1) * 2 + 0) * Ct + v) * ew + col);  // y, last row of strip j-1
        const float z0 = __ldg(sedge + ((int64_t)(j * 2 + 1) * Ct + v) * ew + col);        // z, first row of strip j
        const float e = fmaf(yl, g0, z0) - yl;
        float* X = x + v * plane + col;
        // window row k: k < L is strip j's row k (+= y_last Gamma_j[k]); L <= k < 2L is strip j-1's
        // row HS - 2L + k (+= e Theta_{j-1}[k - L]).  All eight rows are loaded before any is
        // stored (the compiler cannot reorder X loads past X stores on its own).
        float xv[8], pv[8], cv[8];
        int64_t ro[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + u;
            const bool top = k < L;
            ro[u] = top ? (s0 + k) * pitch : (s0 - 2 * L + k) * pitch;
            cv[u] = top ? yl : e;
            if (k < 2 * L) {
                xv[u] = X[ro[u]];
                pv[u] = top ? __ldg(gam + ((int64_t)j * L + k) * pitch + col)
                            : __ldg(theta + ((int64_t)(j - 1) * L + (k - L)) * pitch + col);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k0 + u < 2 * L) X[ro[u]] = fmaf(cv[u], pv[u], xv[u]);
    }
}

cudaError_t launch_seam_fix(float* x, int Ct, const Geometry& g, int HS, int nstrips, int L, const float* gam,
                            const float* theta, const float* sedge, cudaStream_t s) {
    if (nstrips < 2) return cudaSuccess;
    const int ntc = (int)((g.W + 31) / 32);
    return launch_pdl(k_seam_fix, dim3((unsigned)((g.W + 127) / 128), (unsigned)(nstrips - 1), (unsigned)((2 * L + 7) / 8)),
                      dim3(128), 0, s, x, Ct, g.W, g.pitch, g.plane, HS, L, ntc, gam, theta, sedge);
}

// How many rows a carry entering the band keeps an influence >= 2^-26 of itself, maximised
// over the columns (folded into len[0] (top edge) and len[1] (bottom edge) with atomicMax):
// top:    the influence on row k is G_k = prod_{j <= k} a_j (a_0: the link to the band above);
//         rows 0..k-1 need the correction, where k is the first row with G_k < 2^-26;
// bottom: the influence on row H-1-m is Theta = prod_{j = H-m..H} a_j (a_H: the link below).
// The anticausal response Gamma of G is a convex combination of G_m, m >= k, so Gamma_k <= G_k.
// Walks at most Lcap rows per column (d >= 1 bounds the true length by ceil(26 / kc)).
__global__ void k_edge_length(const float* __restrict__ d, int64_t H, int64_t W, int64_t pitch, int Lcap, float kc,
                              unsigned* __restrict__ len) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= W) return;
    const float thr = 1.0f / 67108864.0f;  // 2^-26
    float G = 1.f;
    int k = 0;
    for (; k < Lcap; ++k) {
        G *= coef_from_d(__ldg(d + (int64_t)k * pitch + col), kc);
        if (G < thr) break;
    }
    atomicMax(&len[0], (unsigned)k);
    float Th = 1.f;
    int m = 0;
    for (; m < Lcap; ++m) {
        Th *= coef_from_d(__ldg(d + (H - m) * pitch + col), kc);
        if (Th < thr) break;
    }
    atomicMax(&len[1], (unsigned)m);
}

cudaError_t launch_edge_length(const float* d, const Geometry& g, int Lcap, float kc, unsigned* len, cudaStream_t s) {
    k_edge_length<<<(unsigned)((g.W + 127) / 128), 128, 0, s>>>(d, g.H, g.W, g.pitch, Lcap, kc, len);
    return cudaGetLastError();
}

// the corrections: x[v][k] += c_v Gamma_k (k < L), x[v][k] += e_v Theta_{k-H+L} (k >= H - L), with
// c = y_last of the rank above and e = z_top0 + y_last(this rank) Gamma_0 of the rank below,
// all from the gathered edge records [P][ntiles][2Ct+1][32] (slot 2Ct: Gamma_0)
__global__ void k_edge_fix(float* __restrict__ x, int Ct, int64_t H, int64_t W, int64_t pitch, int64_t plane, int L,
                           const float* __restrict__ gam, const float* __restrict__ theta,
                           const float* __restrict__ gath, int P, int rank, int ntiles, bool cross, bool cut) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int kk = blockIdx.y;  // 0..2L-1: top rows, then bottom rows
    if (col >= W) return;
    const int NT = 2 * Ct + 1;
    const int64_t t = col / colc::TW, cc = col - t * colc::TW;
    const int64_t rstride = (int64_t)ntiles * NT * colc::TW;
    const bool top = kk < L;
    const int64_t row = top ? kk : H - L + (kk - L);
    for (int v = 0; v < Ct; ++v) {
        float carry = 0.f;
        if (top) {
            if (rank > 0) carry = gath[(rank - 1) * rstride + (t * NT + v) * colc::TW + cc];
        } else if (rank + 1 < P) {
            const float* nb = gath + (rank + 1) * rstride + t * NT * colc::TW;
            const float ylast = gath[rank * rstride + (t * NT + v) * colc::TW + cc];
            carry = cross ? fmaf(ylast, nb[(2 * Ct) * colc::TW + cc], nb[(Ct + v) * colc::TW + cc])
                          : nb[(Ct + v) * colc::TW + cc];
            // cut pass (the link below was taken as 0, so z(H-1) = y(H-1)): the missing part is
            // a_H (z_H - y(H-1)), carried upwards by the same Theta
            if (cut) carry -= ylast;
        }
        if (carry != 0.f) {
            const float prof = top ? gam[(int64_t)kk * pitch + col] : theta[(int64_t)(kk - L) * pitch + col];
            float* q = x + v * plane + row * pitch + col;
            *q = fmaf(carry, prof, *q);
        }
    }
}

cudaError_t launch_edge_fix(float* x, int Ct, const Geometry& g, int L, const float* gam, const float* theta,
                            const float* gathered, int P, int rank, cudaStream_t s, bool cross, bool cut) {
    const int ntiles = (int)((g.W + colc::TW - 1) / colc::TW);
    dim3 grid((unsigned)((g.W + 127) / 128), (unsigned)(2 * L));
    k_edge_fix<<<grid, 128, 0, s>>>(x, Ct, g.H, g.W, g.pitch, g.plane, L, gam, theta, gathered, P, rank, ntiles,
                                    cross, cut);
    return cudaGetLastError();
}

}  // namespace dts
