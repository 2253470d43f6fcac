// dts_launch.h -- host-side launchers of the sm_100a kernels (internal to libdts_b200.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dts {

// dts_set_option("pdl"): programmatic dependent launch on the hot-path kernels (default 1)
int option_pdl();
// dts_set_option("row_seg"): forced row-kernel segment length (0 auto; 4, 12, 20, 36)
int option_row_seg();
// launch `kern` on `s` with programmatic stream serialization (see pdl_trigger / pdl_wait)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = option_pdl() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// MODE_TUPLE (cluster column kernel, row-band mode): only the rank band's 5-tuple per column
enum PassMode : int { MODE_FILTER = 0, MODE_UPDATE = 1, MODE_SUPPORT = 2, MODE_ROWUPD = 3, MODE_TUPLE = 4 };
// column-pass phases (row-band mode): FULL = single band set; TUPLE = emit the aggregate
// 5-tuple of this rank's rows; APPLY = finish with external carries (after the exchange)
enum ColPhase : int { PHASE_FULL = 0, PHASE_TUPLE = 1, PHASE_APPLY = 2 };

// Internal planar layout: every H x W plane has row pitch `pitch` floats (a multiple
// of 32, so every row starts 128-B aligned); channel planes are `plane` floats apart.
struct Geometry {
    int64_t H, W, pitch, plane;
};

// K1: domain distances from the HWC guide (Eqs. 8-9; R1, R2).
// a1y (optional): also writes A1 = a_1^{d_y} = 2^(-kc0 d_y), the cluster column kernel's pass-1
// coefficient (north star (1): the derivative kernel writes d and the coefficients a^d)
cudaError_t launch_guide_deriv(const float* guide, int C, float ratio2, const Geometry& g, float* dx, float* dy,
                               cudaStream_t s, float* a1y = nullptr, float kc0 = 0.f);

// K2: recursive-filter row pass (causal + anticausal, fused), FILTER or SUPPORT mode.
struct RowPlan {
    int L, G, R, threads, grid, nbuf;
    size_t smem;
    int64_t rowstride;
    int64_t rowlen = 0;  // floats staged per row (0 / the pitch; a row strip's padded width)
    int minb = 1;        // 2: the two-CTAs-per-SM instantiation (C_t = 3, <= 320 threads)
};
// rowlen > 0: rows of a vertical strip of that (padded) width inside rows of g.pitch
cudaError_t plan_row_pass(const Geometry& g, int Ct, int mode, int num_sms, RowPlan* plan, int64_t rowlen = 0);
// row strips of images wider than one CTA's staging buffer: strip b = columns [c[b], c[b+1])
struct RowStrips {
    int n;
    int c[17];  // c[0] = 0, c[n] = W
};
cudaError_t launch_row_edge_length(const float* d, const Geometry& g, const RowStrips& st, int Lcap, float kc,
                                   unsigned* len, cudaStream_t s);
cudaError_t launch_row_edge_profiles(const float* d, const Geometry& g, const RowStrips& st, int L, float kc,
                                     float* gam, float* theta, bool raw, cudaStream_t s);
// x: row r0 of plane 0 (g.H rows from there); gam / theta: [seam][Hp][L]
cudaError_t launch_row_seam_fix(float* x, int Ct, const Geometry& g, const RowStrips& st, int L, const float* gam,
                                const float* theta, int64_t Hp, int64_t r0, bool raw, cudaStream_t s);
cudaError_t launch_row_pass(const RowPlan& plan, const Geometry& g, int Ct, int mode, const float* in, float* out,
                            const float* d, float kc, cudaStream_t s);

// K2 fused with the previous iteration's Eq. (3) step (MODE_ROWUPD): Z <- Z - step [lam (Z -
// zbar) + chat (Z - T)] written back, then the row filter of the new Z -> out.
struct UpdateArgs;
cudaError_t launch_row_update(const RowPlan& plan, const Geometry& g, int Ct, const float* zbar, float* out,
                              const float* d, float kc, const UpdateArgs& u, cudaStream_t s);

// K3/K4: recursive-filter column pass (decoupled band-tuple scan, cooperative
// persistent grid), FILTER, UPDATE (fused solver step, Eq. 3) or SUPPORT mode.
struct ColPlan {
    int kind;  // 0: decoupled band-tuple kernel (k_col.cu), 1: cluster kernel (k_colc.cu)
    int TW, CB, HB, S, Ls, nb, ntiles, threads;
    int HS = 0, ntc = 0;  // cluster kernel over row strips: strip height, column tiles per strip (0: one strip)
    dim3 grid;
    size_t smem;
    size_t tuple_floats, flag_count;  // scratch the launch needs (ColScratch)
};
struct ColScratch {
    float* tuples;         // >= plan.tuple_floats floats
    unsigned int* flags;   // >= plan.flag_count, zero-initialised once
    unsigned int epoch;    // distinct per launch (flags are compared against it)
    // row-band mode
    int phase;             // ColPhase
    int halo_below;        // the d array has a row H (link to the rank below)
    const float* ext;      // APPLY: [ntiles][2][NV][32] carries into the rank band
    float* rank_tuples;    // TUPLE: [ntiles][2NV+3][32]
};
struct UpdateArgs {
    float* Z;            // planar state (read; written unless out_hwc)
    const float* T;      // planar target
    const float* chat;   // c / S
    float lam, step;
    float* out_hwc;      // when non-null: write the result here (H x W x Ct) instead of Z
    unsigned* resid;     // when non-null (streaming update kernel only): ||g||_inf, atomicMax of float bits
};
cudaError_t plan_col_pass(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan);
cudaError_t launch_col_pass(const ColPlan& plan, const Geometry& g, int Ct, int mode, float* x, const float* d,
                            float kc, const UpdateArgs* upd, float* support, const ColScratch& scr,
                            cudaStream_t s);

// K3/K4 fast path: cluster-held column tiles, register-resident segments (k_colc.cu).
// Returns cudaErrorNotSupported when the shape does not fit (then use plan_col_pass).
cudaError_t plan_col_cluster(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan);
// a row-strip instantiation of the cluster FILTER kernel (A1 input) exists for (C_t, segment rows)
bool colc_strips_supported(int Ct, int ls);
// ls = 16: 16-row warp segments (FILTER, C_t >= 2, not for row bands); plan->Ls records it
// force_cb >= 0: cluster size (0 = auto) instead of the "col_cluster" option
cudaError_t plan_col_cluster_ls(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan, int ls,
                                int force_cb = -1);
cudaError_t launch_col_cluster(const ColPlan& plan, const Geometry& g, int Ct, int mode, float* x, const float* d,
                               float kc, const UpdateArgs* upd, float* support, cudaStream_t s,
                               int nsq = -1,  // nsq >= 0: d holds A1 (see coef_pow)
                               const float* ext = nullptr,    // APPLY: carries into the rank band [ntiles][2][Ct][32]
                               float* rank_tuples = nullptr,   // TUPLE: [ntiles][2Ct+3][32]
                               float* edge = nullptr,          // edge scheme: [ntiles][2Ct+1][32]
                               float* sedge = nullptr,         // row strips: [strip][2][Ct][ntc * 32]
                               float* x_out = nullptr);  // FILTER output planes (null: in place over x)        // row strips: [strip][2][Ct][ntc*32] edge rows

// Eq. (7) confidence: planar X0 = t, X1 = t^2 from a row-major H x W
// target; and, after the DTF of both planes, V = max(0, X1 - X0^2), c = exp(-V / (2 sc^2)).
cudaError_t launch_conf_prologue(const float* target, const Geometry& g, float* X, cudaStream_t s);
cudaError_t launch_conf_epilogue(const float* X, const Geometry& g, float inv_2sc2, float* conf, float* var,
                                 cudaStream_t s);

// Eq. (10) stereo step: Charbonnier target + photometric term, C_t = 1;
// writes Z, or out (H x W) when non-null.
cudaError_t launch_update_stereo(const float* X, float* Z, const float* T, const float* chat, const float* left,
                                 const float* right, int Cg, const Geometry& g, float lam, float step, float gamma,
                                 float eps, float* out, cudaStream_t s);

// Depth-SR front end: bicubic target and bump confidence, (h f) x (w f).
cudaError_t launch_sr_prepare(const float* low, int64_t h, int64_t w, int f, float* target, float* conf,
                              cudaStream_t s);

// dts_set_option("col_cluster") (experiments): forced column-kernel cluster size, 0 = auto
int option_col_cluster();
// dts_set_option("row_two_ctas"): C_t = 3 row passes as two CTAs per SM (k_row.cu)
int row_minb2();

// fill n floats with v
cudaError_t launch_fill(float* p, int64_t n, float v, cudaStream_t s);

// K4b: Eq. (3) update as a streaming kernel (zbar in X); writes Z, or out_hwc when non-null.
// resid (nullable): ||g||_inf of this step folded into *resid as float bits (atomicMax)
cudaError_t launch_update(const float* X, float* Z, const float* T, const float* chat, int Ct, const Geometry& g,
                          float lam, float step, float* out_hwc, int num_sms, cudaStream_t s,
                          unsigned* resid = nullptr);

// compose gathered rank tuples [P][ntiles][2NV+3][32] into this rank's carries
// [ntiles][2][NV][32] (causal carry from the ranks above, anticausal from below)
cudaError_t launch_rank_compose(const float* gathered, int P, int rank, int ntiles, int NV, float* ext,
                                cudaStream_t s);

// K6: solve prologue -- planar Z = T = target, chat = c / S (or c when support_mode = 1).
// Sy (nullable): the column support factor kept separately (S = s_x, chat = c / (S Sy))
cudaError_t launch_prologue(const float* target, const float* conf, int Ct, const Geometry& g, const float* S,
                            const float* Sy,
                            int support_mode, float* Z, float* T, float* chat, cudaStream_t s);

// optional input checks: counts non-finite target/confidence values and confidences outside [0, 1]
cudaError_t launch_check_inputs(const float* target, const float* conf, int Ct, int64_t H, int64_t W,
                                unsigned int* counters, cudaStream_t s);

// Box (normalised-convolution) variant (k_box.cu, reading R25).
// K_B1: fixed-point DT increments q (uint32) to the left / upper neighbour.
cudaError_t launch_box_increments(const float* guide, int C, float k2, const Geometry& g, uint32_t* qx, uint32_t* qy,
                                  cudaStream_t s);
// K_B2: windows of nR - 1 passes (R[0..nR-2]) packed lo | hi << 16 into win planes 2i (rows)
// and 2i + 1 (columns), and the support S = count_x * count_y at R[nR - 1].
cudaError_t launch_box_windows(const uint32_t* qx, const uint32_t* qy, const Geometry& g, const long long* R, int nR,
                               uint32_t* win, float* S, cudaStream_t s);
struct BoxPlan {
    int hx, hy;                                   // halo (max window half-width) per axis
    int row_seg, row_nseg, row_lpad, row_threads, row_grid;
    size_t row_smem;
    int col_seg, col_nseg, col_ntc, col_lpad, col_grid;
    size_t col_smem;
};
cudaError_t plan_box(const Geometry& g, long long R, int num_sms, BoxPlan* plan);
// K_B3 / K_B4: one box pass along rows / columns, in -> out (out of place).
cudaError_t launch_box_row(const BoxPlan& plan, const Geometry& g, int Ct, const float* in, float* out,
                           const uint32_t* win, cudaStream_t s);
cudaError_t launch_box_col(const BoxPlan& plan, const Geometry& g, int Ct, const float* in, float* out,
                           const uint32_t* win, cudaStream_t s);

// Row-band edge fix-up scheme (k_colc.cu): create-time edge profiles of one pass, and the
// elementwise corrections after the gathered edge records.
// raw: keep the causal product profile G (the support's correction) instead of its
// anticausal response Gamma; cross = false: the bottom carry has no causal-carry term
// (the support's P and Q recurrences are independent); cut: the zero-carry pass cut the link
// below the band (z(H-1) = y(H-1)), so the bottom carry is z_H - y(H-1)
cudaError_t launch_edge_profiles(const float* d, const Geometry& g, int L, float kc, float* gam, float* theta,
                                 cudaStream_t s, bool raw = false);
// row-strip seam fix-up of a FILTER column pass run over nstrips strips of HS rows (zero carries
// at each strip's top, link below cut); gam / theta: [nstrips][L][pitch] edge profiles
cudaError_t launch_seam_fix(float* x, int Ct, const Geometry& g, int HS, int nstrips, int L, const float* gam,
                            const float* theta, const float* sedge, cudaStream_t s);
// decay lengths of a band's edge carries (top -> len[0], bottom -> len[1], atomicMax; zero them
// first); d has rows 0..H (row H: the link below the band)
cudaError_t launch_edge_length(const float* d, const Geometry& g, int Lcap, float kc, unsigned* len, cudaStream_t s);
// set cudaFuncAttributeMaxDynamicSharedMemorySize of `fn` on the current device to at least
// `bytes` (tracked per device and function, thread-safe)
cudaError_t ensure_smem_attr(const void* fn, size_t bytes);
cudaError_t launch_edge_fix(float* x, int Ct, const Geometry& g, int L, const float* gam, const float* theta,
                            const float* gathered, int P, int rank, cudaStream_t s, bool cross = true,
                            bool cut = false);

}  // namespace dts
