// dts_capi.cu -- the C ABI declared in include/dts.h: context lifetime, argument
// validation, host/device staging and the per-iteration launch sequence.
//
// Solve loop, for k = 0 .. iterations-1 and passes i = 1..N:
//     K2 row pass i      X <- RF_rows(i == 1 ? Z : X, a_i^{d_x})
//     K3 col pass i      X <- RF_cols(X, a_i^{d_y})                       (i < N)
//     K4 col pass N      Z <- Z - step [lambda (Z - RF_cols(X)) + chat (Z - T)]   (-> out on the last k)
// (readings R4-R12.)
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dts.h"
#include "dts_comm.h"
#include "dts_launch.h"

using namespace dts;

namespace {

thread_local std::string g_last_error;

struct ProfFamily {
    std::string name;
    double bytes_per_launch = 0;
    int64_t launches = 0;
    double total_ms = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};

dts_status cuda_fail(cudaError_t e) {
    g_last_error = cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) return DTS_E_OOM;
    return DTS_E_CUDA;
}

bool finite_pos(float v) { return std::isfinite(v) && v > 0.f; }

enum PtrKind { PTR_DEVICE, PTR_HOST, PTR_BAD };

PtrKind classify(const void* p, int device) {
    if (!p) return PTR_BAD;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return PTR_HOST;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        if (a.type == cudaMemoryTypeDevice && a.device != device) return PTR_BAD;
        return PTR_DEVICE;
    }
    return PTR_HOST;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return pa < pb + nb && pb < pa + na;
}

std::once_flag g_pool_once;

// Process-wide test / experiment options (dts_set_option; include/dts.h).  The defaults are
// the product path; no environment variable changes what the library computes.
struct Options {
    std::atomic<int> col_kernel{0};   // 0: cluster kernel when the column fits, 1: decoupled kernel (k_col.cu)
    std::atomic<int> band_scheme{0};  // 0: edge fix-up when bands are tall enough, 1: TUPLE/APPLY, 2: decoupled
    std::atomic<int> graphs{1};       // replay repeated identical solves as CUDA graphs
    std::atomic<int> row_update{1};   // Eq. (3) step fused into the next iteration's first row pass
    std::atomic<int> col_rows{0};     // column kernel rows per warp segment: 0 auto; 32 or 40 (C_t = 1),
                                      // 12 or 16 (C_t = 3)
    std::atomic<int> col_cluster{0};  // column kernel cluster size: 0 auto, else forced (experiments)
    std::atomic<int> strip_cluster{0};     // row strips: forced cluster size of the strip plan (0 = auto)
    std::atomic<int> band_overlap{1};
    std::atomic<int> row_two_ctas{1};  // C_t = 3 row passes of <= 3840 columns: two CTAs per SM
    std::atomic<int> col_split{0};     // C_t >= 2 column passes: 0 auto (plane by plane over row
                                       // strips), 1 always plane by plane, 2 never
    std::atomic<int> row_seg{0};       // row kernel samples per thread: 0 auto, 4 / 12 / 20 / 36 forced
    std::atomic<int> pdl{1};           // programmatic dependent launch: 0 off, 1 on (trigger at kernel
                                       // end; default), 2 on with the trigger at kernel start  // row bands, edge scheme: all-gather overlapped with the next row pass
    std::atomic<int> col_strips{1};   // tall single-context images: C_t = 1 column passes over row strips
                                      // (0 off, 1 auto, n >= 2: exactly n strips when they fit)
    std::atomic<int> col_oop{1};      // column passes out of place (col_oop): 0 never, 1 row-strip passes,
                                      // 2 every cluster-kernel pass
};
Options& opts_g() {
    static Options o;
    return o;
}

}  // namespace

struct dts_comm {
    dts::Comm* c = nullptr;
};
struct dts_ctx;
extern "C" {  // defined inside the extern "C" section below
static bool strip_plan_n(dts_ctx* ctx, int n, int Ct, ColPlan* out);
static bool batch_strip_plan(dts_ctx* ctx, int Ct, ColPlan* out);
}

// row strips of one image (single GPU; plan_strips / choose_col): n strips of HS rows, per pass
// the measured seam length L and the edge profiles [n][L][pitch], the edge-row buffer
// [n][2][3][ntc * 32] (each strip's last / first output row of up to three planes)
struct StripSet {
    int n = 0, HS = 0;
    std::vector<int> L;
    std::vector<float*> gam, theta;
    float* edge = nullptr;
};

struct dts_ctx {
    int device = 0;
    // row-band mode (multi-GPU): this context owns rows [row0, row0 + g.H) of H_total
    dts::Comm* comm = nullptr;
    int64_t row0 = 0, H_total = 0;
    int halo_above = 0, halo_below = 0;
    float* dx_base = nullptr;  // allocations behind dx / dy (they include the halo rows)
    float* dy_base = nullptr;
    float* rank_tup = nullptr;  // this rank's aggregate tuples   [ntiles][2NV+3][32]
    float* gathered = nullptr;  // all ranks' tuples               [P][ntiles][2NV+3][32]
    float* ext = nullptr;       // carries into this rank's rows   [ntiles][2][NV][32]
    size_t band_cap = 0;
    // edge fix-up scheme, per pass (nullptr: band too short, TUPLE/APPLY instead)
    std::vector<float*> edge_gam, edge_theta;  // L x pitch each: Gamma (top rows), Theta (bottom rows)
    std::vector<int> edge_L;
    // single-GPU row strips for the C_t = 1 FILTER column passes of tall images (DESIGN.md
    // section 7): the cluster plan over strips, per pass the seam length and edge profiles
    std::vector<StripSet*> ssets;  // every strip set built so far (owned)
    StripSet* vs_set = nullptr;    // the create-time C_t = 1 set (plan_strips), or null
    // batched contexts (dts_create_batch): `batch` images of batch_H rows stacked vertically, the
    // column recurrences cut between them (d_y = +inf, A1 = 0 at each image's first row); the
    // FILTER column passes run every image's tiles in one launch (per-C_t strip plan, no seams)
    int64_t batch = 1, batch_H = 0;
    // images wider than the row kernel's staging buffer (plan_row_strips): vertical strips,
    // per pass (and the support, index N) the seam length and the per-row edge profiles
    RowStrips hs{};
    std::vector<int> hs_L;
    std::vector<float*> hs_gam, hs_theta;  // [seam][H][L] each
    ColPlan bs_plan[5]{};
    signed char bs_state[5] = {0, 0, 0, 0, 0};  // 0 not planned, 1 planned, -1 not available
    int num_sms = 148;
    Geometry g{};
    int C = 0;
    float sigma_s = 0, sigma_r = 0;
    int N = 0;
    std::vector<float> kc;  // per pass: sqrt(2) * log2(e) / sigma_i
    float ks = 0;           // support: sqrt(2) * log2(e) / sigma_s
    float* dx = nullptr;
    float* dy = nullptr;
    float* S = nullptr;
    float* Sy = nullptr;  // column support factor when the cluster kernel computes it (S then holds s_x)
    float* A1y = nullptr;  // pass-1 column coefficient a_1^{d_y} (rows 0..H), cluster FILTER passes (N <= 4)
    float* A1y_base = nullptr;  // allocation behind A1y (includes the halo rows, like dy_base)
    // box filter (dts_create_ex, DTS_FILTER_BOX): dx / dy hold the fixed-point increments q,
    // win the packed windows (planes 2i: rows, 2i + 1: columns, pass i), S the window counts
    int filter = DTS_FILTER_RF;
    uint32_t* win = nullptr;
    std::vector<BoxPlan> bplan;
    float* X2 = nullptr;  // second state buffer (box passes are out of place)
    float* Xh = nullptr;  // output planes of out-of-place column passes (col_oop, ensure_xh), xh_cap planes
    int xh_cap = 0;
    bool xh_failed = false;  // Xh could not be allocated: the column passes run in place
    // solver state (allocated for ct_cap target channels)
    int ct_cap = 0;
    float* Z = nullptr;
    float* T = nullptr;
    float* X = nullptr;
    float* chat = nullptr;
    // host staging (device buffers holding host inputs / outputs)
    float* st_t = nullptr;
    float* st_c = nullptr;
    float* st_o = nullptr;
    size_t st_bytes = 0;
    unsigned int* counters = nullptr;
    // column-pass scratch: band tuples + publication flags (epoch-tagged)
    float* tuples = nullptr;
    unsigned int* flags = nullptr;
    size_t tuple_cap = 0, flag_cap = 0;
    unsigned int epoch = 0;
    // CUDA graph of the last solve's launch sequence (cluster column path, device buffers)
    cudaGraphExec_t graph_exec = nullptr;
    std::vector<uintptr_t> graph_key;
    std::vector<uintptr_t> graph_seen;  // key of the last eager solve: a repeat is captured
    int64_t graph_launches = 0;
    cudaStream_t cap_stream = nullptr;
    // row-band edge scheme, overlapped: a FILTER column pass followed by a
    // row pass leaves its all-gather on comm_stream and its edge fix-up pending; the next row
    // pass runs on the band's interior rows first, then waits for the exchange, fixes the L
    // edge rows and filters them
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_cols = nullptr, ev_gath = nullptr;
    struct {
        bool on = false;
        int pass = 0, L = 0, Ct = 0;
        float* x = nullptr;
    } pend;
    // per-iteration ||g||_inf (dts_solve_opts.resid_inf_out), as float bits
    unsigned int* resid = nullptr;
    int resid_cap = 0;
    // row-band mode: scheme decided once at create, identically on every rank (from the
    // all-gathered band heights and carry-decay lengths)
    int64_t band_H_max = 0;
    int band_scheme = 0;  // 0 edge fix-up where the bands allow it, 1 cluster TUPLE/APPLY, 2 decoupled
    cudaStream_t last_stream = nullptr;
    int64_t launches = 0;
};

namespace {

enum Family {
    F_DERIV = 0, F_ROW, F_COL, F_UPDATE, F_SUPPORT_ROW, F_SUPPORT_COL, F_PROLOGUE, F_STEP,
    F_TUPLE, F_EXCHANGE, F_COMPOSE, F_ROWUPD, F_CONF, F_STEREO, F_FILL, F_BOX_PREP, F_BOX_ROW, F_BOX_COL, F_COEF,
    F_SEAM, F_ROWSEAM, F_COUNT
};
const char* kFamilyNames[F_COUNT] = {"guide_deriv", "row_pass", "col_pass", "col_update", "support_row",
                                     "support_col", "prologue", "update", "col_tuple", "exchange",
                                     "rank_compose", "row_update", "confidence", "stereo_update", "link_fill",
                                     "box_windows", "box_row", "box_col", "edge_profiles", "seam_fix",
                                     "row_seam_fix"};

// Process-wide kernel profiler (dts_profile_enable / dts_profile_read): contexts come
// and go inside a timed step, the statistics outlive them.
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<ProfFamily> fam;
    std::vector<cudaEvent_t> pool;
    Profiler() {
        fam.resize(F_COUNT);
        for (int i = 0; i < F_COUNT; ++i) fam[i].name = kFamilyNames[i];
    }
    cudaEvent_t take() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    // resolve pending event pairs (caller synchronised the device)
    void resolve() {
        for (auto& f : fam) {
            for (auto& pr : f.pending) {
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
                    f.total_ms += ms;
                    ++f.launches;
                }
                pool.push_back(pr.first);
                pool.push_back(pr.second);
            }
            f.pending.clear();
        }
    }
};
Profiler& profiler() {
    static Profiler* p = new Profiler();  // never destroyed: events may outlive contexts
    return *p;
}

// Every kernel launch goes through here: counts it and, when profiling, brackets it
// with events on the launch stream.
template <typename F>
dts_status run_launch(dts_ctx* ctx, int fam, double bytes, cudaStream_t s, F&& launch) {
    Profiler& P = profiler();
    const bool prof = P.on;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
        std::lock_guard<std::mutex> lk(P.mu);
        e0 = P.take();
        e1 = P.take();
        cudaEventRecord(e0, s);
    }
    cudaError_t e = launch();
    if (e != cudaSuccess) return cuda_fail(e);
    ++ctx->launches;
    if (prof) {
        std::lock_guard<std::mutex> lk(P.mu);
        cudaEventRecord(e1, s);
        ProfFamily& f = P.fam[fam];
        f.bytes_per_launch = bytes;
        f.pending.emplace_back(e0, e1);
    }
    return DTS_OK;
}

void free_solver_state(dts_ctx* ctx, cudaStream_t s) {
    for (float** p : {&ctx->Z, &ctx->T, &ctx->X, &ctx->chat, &ctx->X2, &ctx->Xh}) {
        if (*p) cudaFreeAsync(*p, s);
        *p = nullptr;
    }
    ctx->ct_cap = 0;
    ctx->xh_cap = 0;
}

dts_status ensure_solver_state(dts_ctx* ctx, int Ct, cudaStream_t s) {
    if (ctx->ct_cap >= Ct && ctx->chat) return DTS_OK;
    free_solver_state(ctx, s);
    const size_t plane = (size_t)ctx->g.plane * sizeof(float);
    cudaError_t e;
    if ((e = cudaMallocAsync((void**)&ctx->Z, plane * Ct, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMallocAsync((void**)&ctx->T, plane * Ct, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMallocAsync((void**)&ctx->X, plane * Ct, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMallocAsync((void**)&ctx->chat, plane, s)) != cudaSuccess) return cuda_fail(e);
    if (ctx->filter == DTS_FILTER_BOX && (e = cudaMallocAsync((void**)&ctx->X2, plane * Ct, s)) != cudaSuccess)
        return cuda_fail(e);
    ctx->ct_cap = Ct;
    return DTS_OK;
}

dts_status ensure_staging(dts_ctx* ctx, size_t bytes_per_image, cudaStream_t s) {
    if (ctx->st_bytes >= bytes_per_image) return DTS_OK;
    for (float** p : {&ctx->st_t, &ctx->st_c, &ctx->st_o}) {
        if (*p) cudaFreeAsync(*p, s);
        *p = nullptr;
    }
    cudaError_t e;
    if ((e = cudaMallocAsync((void**)&ctx->st_t, bytes_per_image, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMallocAsync((void**)&ctx->st_c, bytes_per_image, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMallocAsync((void**)&ctx->st_o, bytes_per_image, s)) != cudaSuccess) return cuda_fail(e);
    ctx->st_bytes = bytes_per_image;
    return DTS_OK;
}

// column-pass plan: cluster fast path when it fits, else the decoupled band-tuple kernel
cudaError_t plan_col(const Geometry& g, int Ct, int mode, int num_sms, ColPlan* plan, int force_cb = -1) {
    if (opts_g().col_kernel.load() == 0) {
        // C_t >= 2 FILTER: 12-row (C_t = 3) or 16-row segments (20 warps per CTA) when the column
        // fits a cluster
        const int rows2 = opts_g().col_rows.load();
        // C_t = 3: 12-row segments (up to 20 warps, grouped segment scans, 96 registers) wherever
        // they plan: batched C3 0.373 against 0.445 ms (16-row), one 4K image 56.0 against 60.3
        // us, one 1080p image 19.0 against 23.0 us
        if (Ct == 3 && mode == MODE_FILTER && rows2 != 16 &&
            plan_col_cluster_ls(g, Ct, mode, num_sms, plan, 12, force_cb) == cudaSuccess)
            return cudaSuccess;
        cudaGetLastError();
        if (Ct >= 2 && mode == MODE_FILTER && rows2 != 12 &&
            plan_col_cluster_ls(g, Ct, mode, num_sms, plan, 16, force_cb) == cudaSuccess) {
            cudaGetLastError();
            return cudaSuccess;
        }
        cudaGetLastError();
        if (plan_col_cluster_ls(g, Ct, mode, num_sms, plan, 32, force_cb) == cudaSuccess) {
            // C_t = 1 FILTER with several tile rounds per launch (throughput-bound): 16 warps
            // x 40-row segments (C4: 0.265 -> 0.249 ms).  One-round images are latency-bound
            // and keep 32-row segments (C1: 12.6 us against 16.8 with 40-row ones).
            const int clusters = (int)(plan->grid.x / plan->CB);
            const int rounds = (plan->ntiles + clusters - 1) / clusters;
            const int rows = opts_g().col_rows.load();
            const bool want40 = rows ? rows == 40 : rounds >= 4;
            ColPlan p40{};
            if (Ct == 1 && mode == MODE_FILTER && want40 &&
                plan_col_cluster_ls(g, Ct, mode, num_sms, &p40, 40, force_cb) == cudaSuccess)
                *plan = p40;
            cudaGetLastError();
            return cudaSuccess;
        }
    }
    cudaGetLastError();
    return plan_col_pass(g, Ct, mode, num_sms, plan);
}

dts_status ensure_col_scratch(dts_ctx* ctx, const ColPlan& cp, cudaStream_t s) {
    cudaError_t e;
    if (cp.kind != 0) return DTS_OK;
    if (cp.tuple_floats > ctx->tuple_cap) {
        if (ctx->tuples) cudaFreeAsync(ctx->tuples, s);
        ctx->tuples = nullptr;
        if ((e = cudaMallocAsync((void**)&ctx->tuples, cp.tuple_floats * sizeof(float), s)) != cudaSuccess)
            return cuda_fail(e);
        ctx->tuple_cap = cp.tuple_floats;
    }
    if (cp.flag_count > ctx->flag_cap) {
        if (ctx->flags) cudaFreeAsync(ctx->flags, s);
        ctx->flags = nullptr;
        if ((e = cudaMallocAsync((void**)&ctx->flags, cp.flag_count * sizeof(unsigned int), s)) != cudaSuccess ||
            (e = cudaMemsetAsync(ctx->flags, 0, cp.flag_count * sizeof(unsigned int), s)) != cudaSuccess)
            return cuda_fail(e);
        ctx->flag_cap = cp.flag_count;
        ctx->epoch = 0;
    }
    return DTS_OK;
}

ColScratch next_scratch(dts_ctx* ctx);

cudaError_t col_launch(dts_ctx* ctx, const ColPlan& plan, int Ct, int mode, float* x, const float* d, float kc,
                       const UpdateArgs* upd, float* support, cudaStream_t s) {
    if (plan.kind == 1) return launch_col_cluster(plan, ctx->g, Ct, mode, x, d, kc, upd, support, s);
    return launch_col_pass(plan, ctx->g, Ct, mode, x, d, kc, upd, support, next_scratch(ctx), s);
}

ColScratch next_scratch(dts_ctx* ctx) {
    ColScratch sc = {};
    sc.phase = PHASE_FULL;
    sc.tuples = ctx->tuples;
    sc.flags = ctx->flags;
    sc.epoch = ++ctx->epoch;
    if (sc.epoch == 0) sc.epoch = ++ctx->epoch;  // flags start at 0: never reuse 0
    return sc;
}

dts_status ensure_band_buffers(dts_ctx* ctx, cudaStream_t s) {
    const int ntiles = (int)((ctx->g.W + 31) / 32);
    const size_t per = (size_t)ntiles * 11 * 32;  // 2NV+3 <= 11 floats per column (NV <= 4)
    if (ctx->band_cap >= per) return DTS_OK;
    cudaError_t e;
    for (float** p : {&ctx->rank_tup, &ctx->gathered, &ctx->ext}) {
        if (*p) cudaFreeAsync(*p, s);
        *p = nullptr;
    }
    if ((e = cudaMallocAsync((void**)&ctx->rank_tup, per * sizeof(float), s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->gathered, per * ctx->comm->nranks * sizeof(float), s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->ext, per * sizeof(float), s)) != cudaSuccess)
        return cuda_fail(e);
    ctx->band_cap = per;
    return DTS_OK;
}

// the pending edge fix-up of an overlapped banded column pass: wait for its exchange, correct
// the L rows at each band edge
static dts_status finish_pending(dts_ctx* ctx, cudaStream_t s) {
    if (!ctx->pend.on) return DTS_OK;
    ctx->pend.on = false;
    cudaError_t e = cudaStreamWaitEvent(s, ctx->ev_gath, 0);
    if (e != cudaSuccess) return cuda_fail(e);
    const int L = ctx->pend.L, Ct = ctx->pend.Ct, pass = ctx->pend.pass;
    float* x = ctx->pend.x;
    return run_launch(ctx, F_COMPOSE, (double)2 * L * ctx->g.W * (8.0 * Ct + 4), s, [&] {
        return launch_edge_fix(x, Ct, ctx->g, L, ctx->edge_gam[pass], ctx->edge_theta[pass], ctx->gathered,
                               ctx->comm->nranks, ctx->comm->rank, s, true, true);
    });
}

// One column pass of a row-band context.  Which scheme runs is
// decided from state every rank shares (the band scheme latched at create from the
// all-gathered band heights and decay lengths, and plans for the TALLEST band), so every
// rank issues the same collective with the same count:
//  - edge fix-up (pass with profiles): zero-carry cluster pass, one all-gather of the edge
//    records, elementwise corrections on L rows at each edge;
//  - cluster TUPLE -> all-gather -> compose -> cluster FILTER with the external carries;
//  - the same on the decoupled kernel (k_col.cu) when the band's columns do not fit a cluster.
dts_status col_pass_banded(dts_ctx* ctx, int Ct, int mode, float* x, float kc, const UpdateArgs* upd,
                           float* support, int fam, double bytes, cudaStream_t s, int pass, bool defer = false) {
    const Geometry& g = ctx->g;
    Geometry gmax = g;  // every rank plans for the tallest band: the same decision everywhere
    gmax.H = ctx->band_H_max;
    gmax.plane = gmax.H * gmax.pitch;
    ColPlan pE, pT, pF;
    const bool edge_ok = ctx->band_scheme == 0 && mode != MODE_SUPPORT && pass >= 0 &&
                         pass < (int)ctx->edge_gam.size() && ctx->edge_gam[pass] &&
                         plan_col(gmax, Ct, MODE_FILTER, ctx->num_sms, &pE) == cudaSuccess && pE.kind == 1;
    cudaGetLastError();
    if (edge_ok && plan_col(g, Ct, MODE_FILTER, ctx->num_sms, &pE) == cudaSuccess && pE.kind == 1) {
        dts_status st;
        cudaError_t e;
        if ((st = ensure_band_buffers(ctx, s)) != DTS_OK) return st;
        const int L = ctx->edge_L[pass];
        const int NT = 2 * Ct + 1;
        const size_t count = (size_t)pE.ntiles * NT * 32;
        const double px = (double)g.H * g.W;
        const bool pre = ctx->A1y && pass < 4;  // pass-1 coefficient squared per pass
        // the single-context kernel with the link below the band cut (a_H taken as 0): its
        // output rows H - 1 and 0 are the exchanged y0(H - 1) and z0(0); the fix-up then
        // carries z_H - y(H - 1) (reading R26)
        st = run_launch(ctx, F_COL, px * (8.0 * Ct + 4), s, [&] {
            return launch_col_cluster(pE, g, Ct, MODE_FILTER, x, pre ? ctx->A1y : ctx->dy, kc, nullptr, nullptr, s,
                                      pre ? pass : -1);  // zero carries
        });
        if (st != DTS_OK) return st;
        for (int v = 0; v < Ct; ++v) {  // y0 at row H - 1 -> slots [0, Ct), z0 at row 0 -> slots [Ct, 2Ct)
            const float* yrow = x + v * g.plane + (g.H - 1) * g.pitch;
            const float* zrow = x + v * g.plane;
            if ((e = cudaMemcpy2DAsync(ctx->rank_tup + v * 32, NT * 32 * sizeof(float), yrow, 32 * sizeof(float),
                                       32 * sizeof(float), pE.ntiles, cudaMemcpyDeviceToDevice, s)) != cudaSuccess ||
                (e = cudaMemcpy2DAsync(ctx->rank_tup + (Ct + v) * 32, NT * 32 * sizeof(float), zrow,
                                       32 * sizeof(float), 32 * sizeof(float), pE.ntiles, cudaMemcpyDeviceToDevice,
                                       s)) != cudaSuccess)
                return cuda_fail(e);
        }
        // Gamma_0 of this rank into slot 2Ct of its records
        if ((e = cudaMemcpy2DAsync(ctx->rank_tup + 2 * Ct * 32, NT * 32 * sizeof(float), ctx->edge_gam[pass],
                                   32 * sizeof(float), 32 * sizeof(float), pE.ntiles, cudaMemcpyDeviceToDevice, s)) !=
            cudaSuccess)
            return cuda_fail(e);
        std::string err;
        // overlapped: the exchange on the context's comm stream, the fix-up left pending for the
        // next row pass (finish_pending)
        const bool ovl = defer && mode == MODE_FILTER && ctx->comm->nranks > 1;
        if (ovl) {
            if ((!ctx->comm_stream &&
                 (e = cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking)) != cudaSuccess) ||
                (!ctx->ev_cols && (e = cudaEventCreateWithFlags(&ctx->ev_cols, cudaEventDisableTiming)) != cudaSuccess) ||
                (!ctx->ev_gath && (e = cudaEventCreateWithFlags(&ctx->ev_gath, cudaEventDisableTiming)) != cudaSuccess) ||
                (e = cudaEventRecord(ctx->ev_cols, s)) != cudaSuccess ||
                (e = cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_cols, 0)) != cudaSuccess)
                return cuda_fail(e);
        }
        cudaStream_t xs = ovl ? ctx->comm_stream : s;
        st = run_launch(ctx, F_EXCHANGE, (double)count * 4 * ctx->comm->nranks, xs, [&] {
            return comm_allgather(ctx->comm, ctx->rank_tup, ctx->gathered, count, xs, &err) ? cudaSuccess
                                                                                             : cudaErrorUnknown;
        });
        if (st != DTS_OK) {
            g_last_error = err;
            return DTS_E_NCCL;
        }
        if (ovl) {
            if ((e = cudaEventRecord(ctx->ev_gath, ctx->comm_stream)) != cudaSuccess) return cuda_fail(e);
            ctx->pend.on = true;
            ctx->pend.pass = pass;
            ctx->pend.L = L;
            ctx->pend.Ct = Ct;
            ctx->pend.x = x;
            return DTS_OK;
        }
        if (ctx->comm->nranks > 1)  // a single rank has no edges to correct
            st = run_launch(ctx, F_COMPOSE, (double)2 * L * g.W * (8.0 * Ct + 4), s, [&] {
                return launch_edge_fix(x, Ct, g, L, ctx->edge_gam[pass], ctx->edge_theta[pass], ctx->gathered,
                                       ctx->comm->nranks, ctx->comm->rank, s, true, true);
            });
        if (st != DTS_OK || mode != MODE_UPDATE) return st;
        return run_launch(ctx, F_STEP, px * (16.0 * Ct + 4), s, [&] {
            return launch_update(x, upd->Z, upd->T, upd->chat, Ct, g, upd->lam, upd->step, upd->out_hwc, ctx->num_sms,
                                 s, upd->resid);
        });
    }
    cudaGetLastError();
    // cluster kernels when the (tallest) band's columns fit a cluster: TUPLE (the rank 5-tuple,
    // with the carry sensitivity as an extra channel) -> all-gather -> compose -> FILTER with
    // the external carries (+ the streaming update kernel for the last pass of an iteration)
    if (mode != MODE_SUPPORT && ctx->band_scheme != 2 &&
        plan_col_cluster(gmax, Ct, MODE_TUPLE, ctx->num_sms, &pT) == cudaSuccess &&
        plan_col_cluster(gmax, Ct, MODE_FILTER, ctx->num_sms, &pF) == cudaSuccess &&
        plan_col_cluster(g, Ct, MODE_TUPLE, ctx->num_sms, &pT) == cudaSuccess &&
        plan_col_cluster(g, Ct, MODE_FILTER, ctx->num_sms, &pF) == cudaSuccess) {
        dts_status st;
        if ((st = ensure_band_buffers(ctx, s)) != DTS_OK) return st;
        const size_t count = (size_t)pF.ntiles * (2 * Ct + 3) * 32;
        const double px = (double)g.H * g.W;
        st = run_launch(ctx, F_TUPLE, px * (4.0 * Ct + 4), s, [&] {
            return launch_col_cluster(pT, g, Ct, MODE_TUPLE, x, ctx->dy, kc, nullptr, nullptr, s, -1, nullptr,
                                      ctx->rank_tup);
        });
        if (st != DTS_OK) return st;
        std::string err;
        st = run_launch(ctx, F_EXCHANGE, (double)count * 4 * ctx->comm->nranks, s, [&] {
            return comm_allgather(ctx->comm, ctx->rank_tup, ctx->gathered, count, s, &err) ? cudaSuccess
                                                                                            : cudaErrorUnknown;
        });
        if (st != DTS_OK) {
            g_last_error = err;
            return DTS_E_NCCL;
        }
        st = run_launch(ctx, F_COMPOSE, 0.0, s, [&] {
            return launch_rank_compose(ctx->gathered, ctx->comm->nranks, ctx->comm->rank, pF.ntiles, Ct, ctx->ext, s);
        });
        if (st != DTS_OK) return st;
        const bool pre = ctx->A1y && pass >= 0 && pass < 4;
        st = run_launch(ctx, F_COL, px * (8.0 * Ct + 4), s, [&] {
            return launch_col_cluster(pF, g, Ct, MODE_FILTER, x, pre ? ctx->A1y : ctx->dy, kc, nullptr, nullptr, s,
                                      pre ? pass : -1, ctx->ext, nullptr);
        });
        if (st != DTS_OK || mode != MODE_UPDATE) return st;
        return run_launch(ctx, F_STEP, px * (16.0 * Ct + 4), s, [&] {
            return launch_update(x, upd->Z, upd->T, upd->chat, Ct, g, upd->lam, upd->step, upd->out_hwc, ctx->num_sms,
                                 s, upd->resid);
        });
    }
    cudaGetLastError();
    ColPlan plan;
    if (plan_col_pass(g, Ct, mode, ctx->num_sms, &plan) != cudaSuccess) return DTS_E_SHAPE;
    dts_status st;
    if ((st = ensure_col_scratch(ctx, plan, s)) != DTS_OK) return st;
    if ((st = ensure_band_buffers(ctx, s)) != DTS_OK) return st;
    const int NV = mode == MODE_SUPPORT ? 1 : Ct;
    const size_t count = (size_t)plan.ntiles * (2 * NV + 3) * 32;
    const double px = (double)g.H * g.W;
    st = run_launch(ctx, F_TUPLE, px * (4.0 * (mode == MODE_SUPPORT ? 0 : NV) + 4), s, [&] {
        ColScratch sc = next_scratch(ctx);
        sc.phase = PHASE_TUPLE;
        sc.halo_below = ctx->halo_below;
        sc.rank_tuples = ctx->rank_tup;
        return launch_col_pass(plan, g, Ct, mode, x, ctx->dy, kc, upd, support, sc, s);
    });
    if (st != DTS_OK) return st;
    std::string err;
    st = run_launch(ctx, F_EXCHANGE, (double)count * 4 * ctx->comm->nranks, s, [&] {
        return comm_allgather(ctx->comm, ctx->rank_tup, ctx->gathered, count, s, &err) ? cudaSuccess
                                                                                        : cudaErrorUnknown;
    });
    if (st != DTS_OK) {
        g_last_error = err;
        return DTS_E_NCCL;
    }
    st = run_launch(ctx, F_COMPOSE, 0.0, s, [&] {
        return launch_rank_compose(ctx->gathered, ctx->comm->nranks, ctx->comm->rank, plan.ntiles, NV, ctx->ext, s);
    });
    if (st != DTS_OK) return st;
    return run_launch(ctx, fam, bytes, s, [&] {
        ColScratch sc = next_scratch(ctx);
        sc.phase = PHASE_APPLY;
        sc.halo_below = ctx->halo_below;
        sc.ext = ctx->ext;
        return launch_col_pass(plan, g, Ct, mode, x, ctx->dy, kc, upd, support, sc, s);
    });
}

// Eager launch, or capture + replay of a CUDA graph: a solve whose key (pointers, sizes,
// scalars) matches the previous eager one is captured on a context-owned stream (the
// caller's may be the uncapturable legacy default stream) and launched as a graph; later
// identical solves replay it.  The launch counter advances as for the eager sequence.
template <typename F>
dts_status run_cached(dts_ctx* ctx, bool use_graph, const std::vector<uintptr_t>& key, cudaStream_t s, F&& enqueue) {
    cudaError_t e;
    dts_status st;
    const bool replay = use_graph && ctx->graph_exec && ctx->graph_key == key;
    const bool capture = use_graph && !replay && ctx->graph_seen == key;
    if (!replay && !capture) {
        if ((st = enqueue(s)) != DTS_OK) return st;
        ctx->graph_seen = use_graph ? key : std::vector<uintptr_t>();
        return DTS_OK;
    }
    if (capture) {
        if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
        ctx->graph_exec = nullptr;
        if (!ctx->cap_stream && (e = cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e);
        cudaStream_t cs = ctx->cap_stream;
        if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return cuda_fail(e);
        const int64_t l0 = ctx->launches;
        st = enqueue(cs);
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(cs, &graph);
        if (st != DTS_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return cuda_fail(e);
        e = cudaGraphInstantiate(&ctx->graph_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            ctx->graph_exec = nullptr;
            return cuda_fail(e);
        }
        ctx->graph_key = key;
        ctx->graph_launches = ctx->launches - l0;
        ctx->launches = l0;
    }
    if ((e = cudaGraphLaunch(ctx->graph_exec, s)) != cudaSuccess) return cuda_fail(e);
    ctx->launches += ctx->graph_launches;
    return DTS_OK;
}

bool profiler_on() {
    Profiler& P = profiler();
    std::lock_guard<std::mutex> lk(P.mu);
    return P.on;
}

}  // namespace

namespace dts {
int option_col_cluster() { return opts_g().col_cluster.load(); }
int row_minb2() { return opts_g().row_two_ctas.load(); }
int option_pdl() { return opts_g().pdl.load(); }
int option_row_seg() { return opts_g().row_seg.load(); }
}  // namespace dts

extern "C" {

const char* dts_version(void) { return "dts-b200 0.2 (sm_100a)"; }

dts_status dts_set_option(const char* name, int32_t value) {
    if (!name) return DTS_E_ARG;
    Options& o = opts_g();
    const std::string n(name);
    if (n == "col_kernel" && (value == 0 || value == 1)) o.col_kernel = value;
    else if (n == "band_scheme" && value >= 0 && value <= 2) o.band_scheme = value;
    else if (n == "graphs" && (value == 0 || value == 1)) o.graphs = value;
    else if (n == "row_update" && (value == 0 || value == 1)) o.row_update = value;
    else if (n == "col_rows" && (value == 0 || value == 12 || value == 16 || value == 32 || value == 40))
        o.col_rows = value;
    else if (n == "col_cluster" && value >= 0 && value <= 16) o.col_cluster = value;
    else if (n == "col_strips" && value >= 0 && value <= 64) o.col_strips = value;
    else if (n == "strip_cluster" && value >= 0 && value <= 16) o.strip_cluster = value;
    else if (n == "col_oop" && value >= 0 && value <= 2) o.col_oop = value;
    else if (n == "band_overlap" && (value == 0 || value == 1)) o.band_overlap = value;
    else if (n == "row_two_ctas" && (value == 0 || value == 1)) o.row_two_ctas = value;
    else if (n == "pdl" && value >= 0 && value <= 2) o.pdl = value;
    else if (n == "col_split" && value >= 0 && value <= 2) o.col_split = value;
    else if (n == "row_seg" && (value == 0 || value == 4 || value == 12 || value == 20 || value == 36))
        o.row_seg = value;
    else return DTS_E_ARG;
    return DTS_OK;
}

// debug hook (not in include/dts.h): the row-strip plan of a context (plan_strips)
int32_t dts_debug_strips(const dts_ctx* ctx, int32_t* HS, int32_t* L3, int32_t* CB, int32_t* grid) {
    if (!ctx) return -1;
    const StripSet* ss = ctx->vs_set;
    ColPlan p{};
    if (ss) strip_plan_n(const_cast<dts_ctx*>(ctx), ss->n, 1, &p);
    if (HS) *HS = ss ? ss->HS : 0;
    for (int i = 0; i < 3 && L3; ++i) L3[i] = ss && i < (int)ss->L.size() ? ss->L[i] : 0;
    if (CB) *CB = ss ? p.CB : 0;
    if (grid) *grid = ss ? (int)p.grid.x : 0;
    return ss ? ss->n : 0;
}

int32_t dts_get_option(const char* name) {
    if (!name) return -1;
    Options& o = opts_g();
    const std::string n(name);
    if (n == "col_kernel") return o.col_kernel;
    if (n == "band_scheme") return o.band_scheme;
    if (n == "graphs") return o.graphs;
    if (n == "row_update") return o.row_update;
    if (n == "col_rows") return o.col_rows;
    if (n == "col_cluster") return o.col_cluster;
    if (n == "col_strips") return o.col_strips;
    if (n == "strip_cluster") return o.strip_cluster;
    if (n == "col_oop") return o.col_oop;
    if (n == "band_overlap") return o.band_overlap;
    if (n == "row_two_ctas") return o.row_two_ctas;
    if (n == "pdl") return o.pdl;
    if (n == "col_split") return o.col_split;
    if (n == "row_seg") return o.row_seg;
    return -1;
}

dts_status dts_sr_prepare(const float* low, int64_t h, int64_t w, int32_t factor, float* target_out,
                          float* conf_out, void* stream) {
    if (!low || !target_out || !conf_out || h < 1 || w < 1 || factor < 1) return DTS_E_ARG;
    const size_t lb = (size_t)h * (size_t)w * sizeof(float);
    const size_t ob = lb * (size_t)factor * (size_t)factor;
    if (overlaps(target_out, ob, low, lb) || overlaps(conf_out, ob, low, lb) || overlaps(target_out, ob, conf_out, ob))
        return DTS_E_ARG;
    int device = 0;
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(e);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const PtrKind kl = classify(low, device), kt = classify(target_out, device), kc = classify(conf_out, device);
    if (kl == PTR_BAD || kt == PTR_BAD || kc == PTR_BAD) return DTS_E_ARG;
    float *dl = nullptr, *dt = nullptr, *dc = nullptr;
    const float* l_d = low;
    float* t_d = target_out;
    float* c_d = conf_out;
    dts_status st = DTS_OK;
    if (kl == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&dl, lb, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(dl, low, lb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            st = cuda_fail(e);
        l_d = dl;
    }
    if (st == DTS_OK && kt == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&dt, ob, s)) != cudaSuccess) st = cuda_fail(e);
        t_d = dt;
    }
    if (st == DTS_OK && kc == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&dc, ob, s)) != cudaSuccess) st = cuda_fail(e);
        c_d = dc;
    }
    if (st == DTS_OK && (e = launch_sr_prepare(l_d, h, w, factor, t_d, c_d, s)) != cudaSuccess) st = cuda_fail(e);
    if (st == DTS_OK && kt == PTR_HOST && (e = cudaMemcpyAsync(target_out, dt, ob, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        st = cuda_fail(e);
    if (st == DTS_OK && kc == PTR_HOST && (e = cudaMemcpyAsync(conf_out, dc, ob, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        st = cuda_fail(e);
    for (float* p : {dl, dt, dc})
        if (p) cudaFreeAsync(p, s);
    if (st == DTS_OK && (kl == PTR_HOST || kt == PTR_HOST || kc == PTR_HOST) &&
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
        st = cuda_fail(e);
    return st;
}

const char* dts_status_string(dts_status s) {
    switch (s) {
        case DTS_OK: return "DTS_OK";
        case DTS_E_ARG: return "DTS_E_ARG: invalid argument";
        case DTS_E_SHAPE: return "DTS_E_SHAPE: unsupported size";
        case DTS_E_NONFINITE: return "DTS_E_NONFINITE: non-finite input";
        case DTS_E_RANGE: return "DTS_E_RANGE: confidence outside [0, 1]";
        case DTS_E_CUDA: return "DTS_E_CUDA: CUDA error";
        case DTS_E_NCCL: return "DTS_E_NCCL: collective error";
        case DTS_E_OOM: return "DTS_E_OOM: out of memory";
    }
    return "unknown dts_status";
}

const char* dts_last_error_string(void) { return g_last_error.c_str(); }

// Wide images: the row kernel stages whole rows of every plane in shared
// memory, which holds 11520 columns at C_t = 4.  Wider images run their row passes over
// vertical strips of at most that width with zero carries at the strip edges, and fix the
// seams up with per-row edge profiles (reading R26 along x): planned here once, from d_x, with
// each pass's (and the support's) measured carry-decay length L, which must fit twice in the
// narrowest strip.
constexpr int64_t kRowStripW = 11520;
static dts_status plan_row_strips(dts_ctx* ctx, cudaStream_t s) {
    const Geometry& g = ctx->g;
    if (g.W <= kRowStripW) return DTS_OK;
    const int n = (int)((g.W + kRowStripW - 1) / kRowStripW);
    if (n > 16) {
        g_last_error = "image too wide (more than 16 row strips)";
        return DTS_E_SHAPE;
    }
    const int64_t WS = ((g.W + n - 1) / n + 31) / 32 * 32;
    RowStrips st{};
    st.n = n;
    for (int b = 0; b < n; ++b) st.c[b] = (int)(b * WS);
    st.c[n] = (int)g.W;
    const int64_t minw = g.W - (int64_t)(n - 1) * WS;
    const int N = ctx->N;
    cudaError_t e;
    unsigned* dlen = nullptr;
    if ((e = cudaMallocAsync((void**)&dlen, 2 * (N + 1) * sizeof(unsigned), s)) != cudaSuccess ||
        (e = cudaMemsetAsync(dlen, 0, 2 * (N + 1) * sizeof(unsigned), s)) != cudaSuccess)
        return cuda_fail(e);
    dts_status st2 = DTS_OK;
    for (int i = 0; i <= N && st2 == DTS_OK; ++i) {
        const float kc = i < N ? ctx->kc[i] : ctx->ks;
        const int Lcap = (int)std::min<int64_t>(std::min<int64_t>((int64_t)std::ceil(26.0 / kc), minw), 1 << 20);
        st2 = run_launch(ctx, F_COEF, (double)g.H * Lcap * 8.0, s,
                         [&] { return launch_row_edge_length(ctx->dx, g, st, Lcap, kc, dlen + 2 * i, s); });
    }
    std::vector<unsigned> len(2 * (N + 1), 0);
    if (st2 == DTS_OK &&
        ((e = cudaMemcpyAsync(len.data(), dlen, len.size() * sizeof(unsigned), cudaMemcpyDeviceToHost, s)) !=
             cudaSuccess ||
         (e = cudaStreamSynchronize(s)) != cudaSuccess))
        st2 = cuda_fail(e);
    cudaFreeAsync(dlen, s);
    if (st2 != DTS_OK) return st2;
    std::vector<int> L(N + 1);
    for (int i = 0; i <= N; ++i) {
        L[i] = (int)std::max<unsigned>(1u, std::max(len[2 * i], len[2 * i + 1]));
        if (2 * (int64_t)L[i] + 1 > minw) {
            g_last_error = "image too wide for row strips at this sigma (a seam correction would overlap)";
            return DTS_E_SHAPE;
        }
    }
    ctx->hs_gam.assign(N + 1, nullptr);
    ctx->hs_theta.assign(N + 1, nullptr);
    for (int i = 0; i <= N && st2 == DTS_OK; ++i) {
        const size_t bytes = (size_t)(n - 1) * g.H * L[i] * sizeof(float);
        if ((e = cudaMallocAsync((void**)&ctx->hs_gam[i], bytes, s)) != cudaSuccess ||
            (e = cudaMallocAsync((void**)&ctx->hs_theta[i], bytes, s)) != cudaSuccess)
            return cuda_fail(e);
        const float kc = i < N ? ctx->kc[i] : ctx->ks;
        st2 = run_launch(ctx, F_COEF, (double)(n - 1) * g.H * L[i] * 12.0, s, [&] {
            return launch_row_edge_profiles(ctx->dx, g, st, L[i], kc, ctx->hs_gam[i], ctx->hs_theta[i], i == N, s);
        });
    }
    if (st2 != DTS_OK) return st2;
    ctx->hs = st;
    ctx->hs_L = L;
    return DTS_OK;
}

// Row pass over rows [r0, r0 + n) of every plane (pass i, or the support when pass < 0; upd:
// the ROWUPD variant with Eq. (3) applied on the fly): one launch when the row fits the
// kernel's staging buffer, else one per row strip and the seam fix-up (plan_row_strips).
static dts_status row_pass_x(dts_ctx* ctx, int Ct, int mode, int pass, const float* in, float* out,
                             const UpdateArgs* upd, int64_t r0, int64_t n, int fam, double bytes, cudaStream_t s) {
    if (n <= 0) return DTS_OK;
    const Geometry& g = ctx->g;
    Geometry gs = g;  // rows r0.. of every plane (the plane stride stays)
    gs.H = n;
    const int64_t o = r0 * g.pitch;
    const float kc = pass >= 0 ? ctx->kc[pass] : ctx->ks;
    const int pmode = upd ? MODE_ROWUPD : (mode == MODE_SUPPORT ? MODE_SUPPORT : MODE_FILTER);
    auto launch = [&](const RowPlan& p, const Geometry& gg, int64_t c0) -> cudaError_t {
        const int64_t oo = o + c0;
        if (upd) {
            UpdateArgs us = *upd;
            us.Z += oo;
            us.T += oo;
            us.chat += oo;
            return launch_row_update(p, gg, Ct, in + oo, out + oo, ctx->dx + oo, kc, us, s);
        }
        return launch_row_pass(p, gg, Ct, mode, in ? in + oo : nullptr, out + oo, ctx->dx + oo, kc, s);
    };
    RowPlan rp{};
    if (plan_row_pass(gs, Ct, pmode, ctx->num_sms, &rp) == cudaSuccess)
        return run_launch(ctx, fam, bytes, s, [&] { return launch(rp, gs, 0); });
    cudaGetLastError();
    const RowStrips& st = ctx->hs;
    if (st.n < 2) return DTS_E_SHAPE;
    for (int b = 0; b < st.n; ++b) {
        Geometry gb = gs;
        gb.W = st.c[b + 1] - st.c[b];
        RowPlan pb{};
        if (plan_row_pass(gb, Ct, pmode, ctx->num_sms, &pb, (gb.W + 3) / 4 * 4) != cudaSuccess) return DTS_E_SHAPE;
        const dts_status r = run_launch(ctx, fam, bytes * (double)gb.W / (double)g.W, s,
                                        [&] { return launch(pb, gb, st.c[b]); });
        if (r != DTS_OK) return r;
    }
    const int li = pass >= 0 ? pass : ctx->N;
    const int L = ctx->hs_L[li];
    const int planes = mode == MODE_SUPPORT ? 1 : Ct;
    return run_launch(ctx, F_ROWSEAM, (double)(st.n - 1) * n * 2 * L * 12.0 * planes, s, [&] {
        return launch_row_seam_fix(out + o, planes, gs, st, L, ctx->hs_gam[li], ctx->hs_theta[li], g.H, r0,
                                   mode == MODE_SUPPORT, s);
    });
}

// Tall single-context images: a column tile must sit on chip across its
// cluster, and the clusters a tall column needs (16 CTAs for C4) pack only 7 per GPU (112 of
// 148 SMs); columns taller than 16 CTAs hold do not fit a cluster at all.  Cut the image into
// row strips whose columns fit smaller clusters, run the FILTER passes over all strips in one
// launch (zero carry at each strip's top, link below cut) and add the carries at the seams
// afterwards (k_seam_fix, reading R26).  A strip set (n strips) holds every pass's measured
// carry-decay length L (k_edge_length: influence below 2^-26 after L rows), which must fit
// twice in the shortest strip, the edge profiles and the edge-row buffer; its per-C_t plans
// are made on use.

// the plan over n strips for C_t (a strip column must fit a cluster)
static bool strip_plan_n(dts_ctx* ctx, int n, int Ct, ColPlan* out) {
    const Geometry& g = ctx->g;
    const int64_t HS = (g.H + n - 1) / n;
    if (n < 2 || HS < 64 || (int64_t)(n - 1) * HS >= g.H) return false;
    Geometry gs = g;  // planned as n strips side by side: the launch has n times the tiles
    gs.H = HS;
    gs.W = g.W * n;
    gs.pitch = (gs.W + 31) / 32 * 32;
    gs.plane = HS * gs.pitch;
    ColPlan ps{};
    const bool ok = gs.W <= ((int64_t)1 << 31) / 2 &&
                    plan_col(gs, Ct, MODE_FILTER, ctx->num_sms, &ps, opts_g().strip_cluster.load()) == cudaSuccess &&
                    ps.kind == 1 && colc_strips_supported(Ct, ps.Ls);
    cudaGetLastError();
    if (!ok) return false;
    ps.HS = (int)HS;
    ps.ntc = (int)((g.W + 31) / 32);
    ps.ntiles = ps.ntc * n;
    *out = ps;
    return true;
}

// measure the seam lengths of n strips and build their profiles (syncs s once); *out stays
// null when a seam correction would overlap the next (2L + 1 > the last strip)
static dts_status build_strip_set(dts_ctx* ctx, int n, cudaStream_t s, StripSet** out) {
    *out = nullptr;
    const Geometry& g = ctx->g;
    const int HS = (int)((g.H + n - 1) / n);
    const int64_t Hlast = g.H - (int64_t)(n - 1) * HS;
    const int N = ctx->N;
    cudaError_t e;
    unsigned* dlen = nullptr;
    if ((e = cudaMallocAsync((void**)&dlen, 2 * N * sizeof(unsigned), s)) != cudaSuccess ||
        (e = cudaMemsetAsync(dlen, 0, 2 * N * sizeof(unsigned), s)) != cudaSuccess)
        return cuda_fail(e);
    dts_status st = DTS_OK;
    for (int i = 0; i < N && st == DTS_OK; ++i) {
        const int64_t worst = (int64_t)std::ceil(26.0 / (double)ctx->kc[i]);
        const int Lcap = (int)std::min<int64_t>(std::min<int64_t>(worst, Hlast), 1 << 20);
        for (int b = 0; b < n && st == DTS_OK; ++b) {
            Geometry gs = g;
            gs.H = std::min<int64_t>(HS, g.H - (int64_t)b * HS);
            st = run_launch(ctx, F_COEF, (double)g.W * Lcap * 8.0, s, [&] {
                return launch_edge_length(ctx->dy + (int64_t)b * HS * g.pitch, gs, Lcap, ctx->kc[i], dlen + 2 * i, s);
            });
        }
    }
    std::vector<unsigned> len(2 * N, 0);
    if (st == DTS_OK && ((e = cudaMemcpyAsync(len.data(), dlen, 2 * N * sizeof(unsigned), cudaMemcpyDeviceToHost, s)) !=
                             cudaSuccess ||
                         (e = cudaStreamSynchronize(s)) != cudaSuccess))
        st = cuda_fail(e);
    cudaFreeAsync(dlen, s);
    if (st != DTS_OK) return st;
    std::vector<int> L(N);
    for (int i = 0; i < N; ++i) {
        L[i] = (int)std::max<unsigned>(1u, std::max(len[2 * i], len[2 * i + 1]));
        if (2 * (int64_t)L[i] + 1 > Hlast) return DTS_OK;  // a seam correction would overlap
    }
    StripSet* ss = new StripSet();
    ss->n = n;
    ss->HS = HS;
    ss->L = L;
    ctx->ssets.push_back(ss);  // owned by the context from here on (dts_destroy frees it)
    ss->gam.assign(N, nullptr);
    ss->theta.assign(N, nullptr);
    for (int i = 0; i < N && st == DTS_OK; ++i) {
        const size_t bytes = (size_t)n * L[i] * g.pitch * sizeof(float);
        if ((e = cudaMallocAsync((void**)&ss->gam[i], bytes, s)) != cudaSuccess ||
            (e = cudaMallocAsync((void**)&ss->theta[i], bytes, s)) != cudaSuccess)
            return cuda_fail(e);
        for (int b = 0; b < n && st == DTS_OK; ++b) {
            Geometry gs = g;
            gs.H = std::min<int64_t>(HS, g.H - (int64_t)b * HS);
            st = run_launch(ctx, F_COEF, (double)g.W * 2 * L[i] * 12.0, s, [&] {
                return launch_edge_profiles(ctx->dy + (int64_t)b * HS * g.pitch, gs, L[i], ctx->kc[i],
                                            ss->gam[i] + (size_t)b * L[i] * g.pitch,
                                            ss->theta[i] + (size_t)b * L[i] * g.pitch, s);
            });
        }
    }
    if (st != DTS_OK) return st;
    // edge rows of up to C_t = 3 planes (the cluster kernel's widest)
    if ((e = cudaMallocAsync((void**)&ss->edge, (size_t)n * 2 * 3 * ((g.W + 31) / 32) * 32 * sizeof(float), s)) !=
        cudaSuccess)
        return cuda_fail(e);
    *out = ss;
    return DTS_OK;
}

static StripSet* find_strip_set(dts_ctx* ctx, int n) {
    for (StripSet* ss : ctx->ssets)
        if (ss->n == n) return ss;
    return nullptr;
}

// create time, C_t = 1: strips for columns that fit a cluster but need big clusters (GPC
// packing wastes SMs) and several tile rounds per launch (throughput-bound; small images stay
// latency-bound and keep one strip).  Preference (measured on C4, unprofiled 20-iteration
// solves, tools/strips4.sh): the fewest strips whose plan covers >= 90% of the SMs and adds
// >= 10% over one strip (C4: 2 strips of 5000 rows on 15 clusters of 9, 30.58 ms against 31.18
// unstripped; 4 strips x clusters of 4 30.84; 16 strips x 2 CTAs of 320 rows per SM 31.33 -- its
// column kernel is the fastest, 0.204 ms, but 15 seams cost more than that saves).  Columns
// too tall for one cluster get their strips per C_t at the first solve (choose_col).
static dts_status plan_strips(dts_ctx* ctx, cudaStream_t s) {
    const Geometry& g = ctx->g;
    ColPlan base{};
    if (plan_col(g, 1, MODE_FILTER, ctx->num_sms, &base) != cudaSuccess || base.kind != 1) {
        cudaGetLastError();
        return DTS_OK;
    }
    const int forced = opts_g().col_strips.load();
    const int rounds = base.ntiles * base.CB / (int)base.grid.x;
    if (forced < 2 && (base.CB < 8 || rounds < 4)) return DTS_OK;
    int best_n = 0;
    for (int n : {2, 4, 8, 16, 32}) {
        if (forced >= 2 && n != forced) continue;
        ColPlan ps{};
        if (!strip_plan_n(ctx, n, 1, &ps)) {
            if ((g.H + n - 1) / n < 64) break;
            continue;
        }
        const bool wide = ps.grid.x * 10 >= (unsigned)ctx->num_sms * 9 && ps.grid.x * 10 >= base.grid.x * 11;
        if (wide || forced >= 2) {
            best_n = n;
            break;
        }
    }
    if (!best_n) return DTS_OK;
    StripSet* ss = nullptr;
    dts_status st = build_strip_set(ctx, best_n, s, &ss);
    if (st == DTS_OK && ss) ctx->vs_set = ss;
    return st;
}

// Row-band contexts: every rank measures how many rows a carry
// entering its band edges keeps an influence >= 2^-26 of itself (per pass, and for the
// support), from its own coefficients; the ranks all-gather (rows, lengths) and every rank
// takes the same decisions from the same numbers: L_i = the largest length over ranks and
// edges, the edge fix-up scheme for pass i iff the SHORTEST band holds 2 L_i + 1 rows.
// Lengths: [0, N) the passes, N the support.  Returns the agreed lengths (0: no edge scheme).
static dts_status band_agree(dts_ctx* ctx, cudaStream_t s, std::vector<int>* L_agreed) {
    dts::Comm* comm = ctx->comm;
    const int N = ctx->N, nl = N + 1, P = comm->nranks;
    const int rec = 2 + 2 * nl;  // [rows, 0, (top, bottom) x nl] as 32-bit words
    unsigned* dlen = nullptr;
    float *send = nullptr, *recv = nullptr;
    cudaError_t e;
    dts_status st = DTS_OK;
    std::vector<unsigned> host(rec, 0u), all((size_t)rec * P, 0u);
    auto cleanup = [&]() {
        for (void* q : {(void*)dlen, (void*)send, (void*)recv})
            if (q) cudaFreeAsync(q, s);
    };
    if ((e = cudaMallocAsync((void**)&dlen, 2 * nl * sizeof(unsigned), s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&send, rec * sizeof(float), s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&recv, (size_t)rec * P * sizeof(float), s)) != cudaSuccess ||
        (e = cudaMemsetAsync(dlen, 0, 2 * nl * sizeof(unsigned), s)) != cudaSuccess) {
        cleanup();
        return cuda_fail(e);
    }
    for (int i = 0; i < nl && st == DTS_OK; ++i) {
        const float kc = i < N ? ctx->kc[i] : ctx->ks;  // coefficient 2^(-kc d), d >= 1
        const int64_t worst = (int64_t)std::ceil(26.0 / (double)kc);
        const int Lcap = (int)std::min<int64_t>(std::min<int64_t>(worst, ctx->g.H), 1 << 20);
        st = run_launch(ctx, F_COEF, (double)ctx->g.W * Lcap * 8.0, s,
                        [&] { return launch_edge_length(ctx->dy, ctx->g, Lcap, kc, dlen + 2 * i, s); });
    }
    if (st == DTS_OK &&
        ((e = cudaMemcpyAsync(host.data() + 2, dlen, 2 * nl * sizeof(unsigned), cudaMemcpyDeviceToHost, s)) !=
             cudaSuccess ||
         (e = cudaStreamSynchronize(s)) != cudaSuccess))
        st = cuda_fail(e);
    host[0] = (unsigned)ctx->g.H;
    if (st == DTS_OK && (e = cudaMemcpyAsync(send, host.data(), rec * sizeof(unsigned), cudaMemcpyHostToDevice, s)) !=
                            cudaSuccess)
        st = cuda_fail(e);
    std::string err;
    if (st == DTS_OK) {  // the words travel as opaque 32-bit values
        st = run_launch(ctx, F_EXCHANGE, (double)rec * 4 * P, s, [&] {
            return comm_allgather(comm, send, recv, (size_t)rec, s, &err) ? cudaSuccess : cudaErrorUnknown;
        });
        if (st != DTS_OK && !err.empty()) {
            g_last_error = err;
            st = DTS_E_NCCL;
        }
    }
    if (st == DTS_OK &&
        ((e = cudaMemcpyAsync(all.data(), recv, (size_t)rec * P * sizeof(unsigned), cudaMemcpyDeviceToHost, s)) !=
             cudaSuccess ||
         (e = cudaStreamSynchronize(s)) != cudaSuccess))
        st = cuda_fail(e);
    cleanup();
    if (st != DTS_OK) return st;
    int64_t hmin = INT64_MAX, hmax = 0;
    for (int r = 0; r < P; ++r) {
        hmin = std::min<int64_t>(hmin, all[(size_t)r * rec]);
        hmax = std::max<int64_t>(hmax, all[(size_t)r * rec]);
    }
    ctx->band_H_max = hmax;
    L_agreed->assign(nl, 0);
    for (int i = 0; i < nl; ++i) {
        int64_t L = 1;
        for (int r = 0; r < P; ++r)
            for (int edge = 0; edge < 2; ++edge) L = std::max<int64_t>(L, all[(size_t)r * rec + 2 + 2 * i + edge]);
        (*L_agreed)[i] = (ctx->band_scheme == 0 && 2 * L + 1 <= hmin && L <= (1 << 20)) ? (int)L : 0;
    }
    return DTS_OK;
}

static dts_status create_impl(const float* guide, int64_t H_total, int64_t row0, int64_t H, int64_t W, int32_t C,
                              float sigma_s, float sigma_r, int32_t filter_passes, dts::Comm* comm, void* stream,
                              dts_ctx** out_ctx, int64_t batch = 1) {
    if (!out_ctx || !guide) return DTS_E_ARG;
    *out_ctx = nullptr;
    if (H < 1 || W < 1 || C < 1) return DTS_E_ARG;
    if (row0 < 0 || row0 + H > H_total) return DTS_E_ARG;
    if (!comm && (row0 != 0 || H != H_total)) return DTS_E_ARG;
    if (batch < 1 || H % batch != 0 || (comm && batch != 1)) return DTS_E_ARG;
    if (!finite_pos(sigma_s) || !finite_pos(sigma_r)) return DTS_E_ARG;
    if (filter_passes < 1 || filter_passes > 16) return DTS_E_ARG;
    if (W > 16 * kRowStripW || H > (int64_t)1 << 30 || C > 4096) return DTS_E_SHAPE;
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    int device = 0;
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(e);
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major < 10) {
        g_last_error = "device is not sm_100-class";
        return DTS_E_CUDA;
    }
    std::call_once(g_pool_once, [device]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;  // keep freed blocks cached: create/destroy cycles do not hit the driver
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });

    dts_ctx* ctx = new dts_ctx();
    ctx->device = device;
    ctx->comm = comm;
    ctx->row0 = row0;
    ctx->H_total = H_total;
    ctx->batch = batch;
    ctx->batch_H = H / batch;
    ctx->halo_above = row0 > 0 ? 1 : 0;
    ctx->halo_below = row0 + H < H_total ? 1 : 0;
    const int64_t Hx = H + ctx->halo_above + ctx->halo_below;  // guide rows passed in
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    ctx->g.H = H;
    ctx->g.W = W;
    ctx->g.pitch = (W + 31) / 32 * 32;
    ctx->g.plane = H * ctx->g.pitch;
    ctx->C = C;
    ctx->sigma_s = sigma_s;
    ctx->sigma_r = sigma_r;
    ctx->N = filter_passes;
    // R5: sigma_i = sigma_s sqrt(3) 2^(N-i) / sqrt(4^N - 1); coefficient a_i^d = 2^(-kc_i d)
    const double log2e = 1.4426950408889634, sqrt2 = 1.4142135623730951;
    const double denom = std::sqrt(std::pow(4.0, filter_passes) - 1.0);
    for (int i = 1; i <= filter_passes; ++i) {
        const double sig = sigma_s * std::sqrt(3.0) * std::pow(2.0, filter_passes - i) / denom;
        ctx->kc.push_back((float)(sqrt2 * log2e / sig));
    }
    ctx->ks = (float)(sqrt2 * log2e / sigma_s);

    // plans (validate that this build supports the shape before allocating)
    RowPlan rp;
    ColPlan cp;
    // rows wider than the row kernel stages run over row strips (plan_row_strips, below)
    if ((plan_row_pass(ctx->g, 1, MODE_SUPPORT, ctx->num_sms, &rp) != cudaSuccess && W <= kRowStripW) ||
        (comm ? plan_col_pass(ctx->g, 1, MODE_SUPPORT, ctx->num_sms, &cp)
              : plan_col(ctx->g, 1, MODE_SUPPORT, ctx->num_sms, &cp)) != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return DTS_E_SHAPE;
    }
    cudaGetLastError();

    const size_t plane = (size_t)ctx->g.plane * sizeof(float);
    dts_status st = DTS_OK;
    const float* gdev = guide;
    float* gstage = nullptr;
    PtrKind gk = classify(guide, device);
    if (gk == PTR_BAD) {
        delete ctx;
        return DTS_E_ARG;
    }
    const size_t plane_x = (size_t)Hx * ctx->g.pitch * sizeof(float);
    // d_y gets one extra row: row H of the band is the link to the rows below (the halo
    // when there is one, else +inf: A = 0 at the image bottom, R4) -- the streaming
    // column kernel reads it as the band-closing coefficient
    if ((e = cudaMallocAsync((void**)&ctx->dx_base, plane_x, s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->dy_base, plane_x + ctx->g.pitch * sizeof(float), s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->S, plane, s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->counters, 2 * sizeof(unsigned int), s)) != cudaSuccess) {
        st = cuda_fail(e);
        dts_destroy(ctx);
        return st;
    }
    ctx->dx = ctx->dx_base + ctx->halo_above * ctx->g.pitch;
    ctx->dy = ctx->dy_base + ctx->halo_above * ctx->g.pitch;
    const size_t gbytes = (size_t)Hx * W * C * sizeof(float);
    if (gk == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&gstage, gbytes, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(gstage, guide, gbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
            st = cuda_fail(e);
            if (gstage) cudaFreeAsync(gstage, s);
            dts_destroy(ctx);
            return st;
        }
        gdev = gstage;
    }
    const float ratio = sigma_s / sigma_r;
    const double px = (double)H * W;
    Geometry gx = ctx->g;  // the guide rows including halos
    gx.H = Hx;
    gx.plane = Hx * gx.pitch;
    // the cluster column kernel reads a_1^{d_y} instead of d_y (one exp per pixel, written by
    // the derivative kernel, instead of one per pixel and pass); later passes square it (R5:
    // sigma halves per pass).  Rows 0..H: row H is the bottom link (+inf -> 0).
    const bool with_a1 = filter_passes <= 4;  // every cluster column pass reads it (full height or strips)
    if (with_a1 && (e = cudaMallocAsync((void**)&ctx->A1y_base, (size_t)(Hx + 1) * ctx->g.pitch * sizeof(float), s)) !=
                       cudaSuccess) {
        st = cuda_fail(e);
        if (gstage) cudaFreeAsync(gstage, s);
        dts_destroy(ctx);
        return st;
    }
    if (ctx->A1y_base) ctx->A1y = ctx->A1y_base + ctx->halo_above * ctx->g.pitch;
    st = run_launch(ctx, F_DERIV, px * (4.0 * C + 8.0 + (with_a1 ? 4.0 : 0.0)), s, [&] {
        return launch_guide_deriv(gdev, C, ratio * ratio, gx, ctx->dx_base, ctx->dy_base, s, ctx->A1y_base,
                                  ctx->kc[0]);
    });
    if (st == DTS_OK && !ctx->halo_below) {
        const float inf = std::numeric_limits<float>::infinity();
        st = run_launch(ctx, F_FILL, ctx->g.pitch * 4.0, s,
                        [&] { return launch_fill(ctx->dy + H * ctx->g.pitch, ctx->g.pitch, inf, s); });
        if (st == DTS_OK && ctx->A1y)
            st = run_launch(ctx, F_FILL, ctx->g.pitch * 4.0, s,
                            [&] { return launch_fill(ctx->A1y + H * ctx->g.pitch, ctx->g.pitch, 0.f, s); });
    }
    // batched contexts: cut the column links between the stacked images (R4 at each image's
    // first row: d_y = +inf, A = 0), so that every recurrence restarts there exactly
    for (int64_t b = 1; b < batch && st == DTS_OK; ++b) {
        const float inf = std::numeric_limits<float>::infinity();
        const int64_t r = b * ctx->batch_H;
        st = run_launch(ctx, F_FILL, ctx->g.pitch * 4.0, s,
                        [&] { return launch_fill(ctx->dy + r * ctx->g.pitch, ctx->g.pitch, inf, s); });
        if (st == DTS_OK && ctx->A1y)
            st = run_launch(ctx, F_FILL, ctx->g.pitch * 4.0, s,
                            [&] { return launch_fill(ctx->A1y + r * ctx->g.pitch, ctx->g.pitch, 0.f, s); });
    }
    if (st == DTS_OK) st = plan_row_strips(ctx, s);
    if (st == DTS_OK)
        st = row_pass_x(ctx, 1, MODE_SUPPORT, -1, nullptr, ctx->S, nullptr, 0, H, F_SUPPORT_ROW, px * 8.0, s);
    if (st == DTS_OK) st = ensure_col_scratch(ctx, cp, s);
    Geometry gi = ctx->g;  // one image of a batched context
    gi.H = ctx->batch_H;
    gi.plane = gi.H * gi.pitch;
    ColPlan cpi{};
    const bool per_image_support = batch > 1 && cp.kind != 1 &&
                                   plan_col(gi, 1, MODE_SUPPORT, ctx->num_sms, &cpi) == cudaSuccess && cpi.kind == 1;
    cudaGetLastError();
    std::vector<int> band_L;  // agreed edge lengths (row-band contexts): passes, then the support
    if (st == DTS_OK && comm) {
        ctx->band_scheme = opts_g().band_scheme.load();  // latched: the same on every rank of a job
        st = band_agree(ctx, s, &band_L);
    }
    if (st == DTS_OK) {
        if (comm) {
            // edge scheme for the support: s = P + Q - 1 with independent
            // causal P and anticausal Q; the zero-carry cluster pass gives s0 with P0(0) = 1 and
            // Q0(H-1) = 1, so s0(H-1) is the P carry for the rank below and s0(0) the Q carry for
            // the rank above; then s += c G_k (top rows) + e Theta_k (bottom rows)
            const int64_t Ls = band_L[filter_passes];
            Geometry gmax = ctx->g;  // decided for the tallest band: the same on every rank
            gmax.H = ctx->band_H_max;
            gmax.plane = gmax.H * gmax.pitch;
            ColPlan cps;
            bool edge = Ls >= 1 && plan_col_cluster(gmax, 1, MODE_SUPPORT, ctx->num_sms, &cps) == cudaSuccess &&
                        plan_col_cluster(ctx->g, 1, MODE_SUPPORT, ctx->num_sms, &cps) == cudaSuccess;
            cudaGetLastError();
            if (edge) {
                float *G = nullptr, *Th = nullptr;
                const size_t pb = (size_t)Ls * ctx->g.pitch * sizeof(float);
                if ((e = cudaMallocAsync((void**)&ctx->Sy, plane, s)) != cudaSuccess ||
                    (e = cudaMallocAsync((void**)&G, pb, s)) != cudaSuccess ||
                    (e = cudaMallocAsync((void**)&Th, pb, s)) != cudaSuccess)
                    st = cuda_fail(e);
                if (st == DTS_OK) st = ensure_band_buffers(ctx, s);
                if (st == DTS_OK)
                    st = run_launch(ctx, F_SUPPORT_COL, px * 8.0, s, [&] {
                        return launch_col_cluster(cps, ctx->g, 1, MODE_SUPPORT, nullptr, ctx->dy, ctx->ks, nullptr,
                                                  ctx->Sy, s);
                    });
                const int NT = 3;
                const size_t count = (size_t)cps.ntiles * NT * 32;
                if (st == DTS_OK &&
                    ((e = cudaMemsetAsync(ctx->rank_tup, 0, count * sizeof(float), s)) != cudaSuccess ||
                     (e = cudaMemcpy2DAsync(ctx->rank_tup, NT * 32 * sizeof(float), ctx->Sy + (H - 1) * ctx->g.pitch,
                                            32 * sizeof(float), 32 * sizeof(float), cps.ntiles,
                                            cudaMemcpyDeviceToDevice, s)) != cudaSuccess ||
                     (e = cudaMemcpy2DAsync(ctx->rank_tup + 32, NT * 32 * sizeof(float), ctx->Sy, 32 * sizeof(float),
                                            32 * sizeof(float), cps.ntiles, cudaMemcpyDeviceToDevice, s)) !=
                         cudaSuccess))
                    st = cuda_fail(e);
                std::string err;
                if (st == DTS_OK)
                    st = run_launch(ctx, F_EXCHANGE, (double)count * 4 * comm->nranks, s, [&] {
                        return comm_allgather(comm, ctx->rank_tup, ctx->gathered, count, s, &err) ? cudaSuccess
                                                                                                  : cudaErrorUnknown;
                    });
                if (st == DTS_E_CUDA && !err.empty()) {
                    g_last_error = err;
                    st = DTS_E_NCCL;
                }
                if (st == DTS_OK)
                    st = run_launch(ctx, F_COEF, px * 8.0, s, [&] {
                        return launch_edge_profiles(ctx->dy, ctx->g, (int)Ls, ctx->ks, G, Th, s, true);
                    });
                if (st == DTS_OK && comm->nranks > 1)
                    st = run_launch(ctx, F_COMPOSE, (double)2 * Ls * W * 12.0, s, [&] {
                        return launch_edge_fix(ctx->Sy, 1, ctx->g, (int)Ls, G, Th, ctx->gathered, comm->nranks,
                                               comm->rank, s, false);
                    });
                if (G) cudaFreeAsync(G, s);
                if (Th) cudaFreeAsync(Th, s);
            } else {
                st = col_pass_banded(ctx, 1, MODE_SUPPORT, nullptr, ctx->ks, nullptr, ctx->S, F_SUPPORT_COL,
                                     px * 12.0, s, -1);
            }
        } else if (per_image_support) {
            // batched context too tall for one cluster column: s_y image by image on the cluster
            // kernel (each image's column ends at the cut below it)
            if ((e = cudaMallocAsync((void**)&ctx->Sy, plane, s)) != cudaSuccess) st = cuda_fail(e);
            for (int64_t b = 0; b < batch && st == DTS_OK; ++b) {
                const int64_t off = b * ctx->batch_H * ctx->g.pitch;
                st = run_launch(ctx, F_SUPPORT_COL, (double)gi.H * W * 8.0, s, [&] {
                    return launch_col_cluster(cpi, gi, 1, MODE_SUPPORT, nullptr, ctx->dy + off, ctx->ks, nullptr,
                                              ctx->Sy + off, s);
                });
            }
        } else if (cp.kind == 1) {  // cluster kernel: s_y into its own plane (no read-modify-write of S)
            if ((e = cudaMallocAsync((void**)&ctx->Sy, plane, s)) != cudaSuccess) st = cuda_fail(e);
            if (st == DTS_OK)
                st = run_launch(ctx, F_SUPPORT_COL, px * 8.0, s, [&] {
                    return col_launch(ctx, cp, 1, MODE_SUPPORT, nullptr, ctx->dy, ctx->ks, nullptr, ctx->Sy, s);
                });
        } else {
            st = run_launch(ctx, F_SUPPORT_COL, px * 12.0, s, [&] {
                return col_launch(ctx, cp, 1, MODE_SUPPORT, nullptr, ctx->dy, ctx->ks, nullptr, ctx->S, s);
            });
        }
    }
    // row-band contexts: edge profiles of every pass whose agreed edge length L (carry
    // influence < 2^-26 after L rows, measured on every rank) fits twice in the shortest band
    if (st == DTS_OK && comm) {
        ctx->edge_gam.assign(filter_passes, nullptr);
        ctx->edge_theta.assign(filter_passes, nullptr);
        ctx->edge_L.assign(filter_passes, 0);
        for (int i = 1; i <= filter_passes && st == DTS_OK; ++i) {
            const int64_t L = band_L[i - 1];
            if (L < 1) continue;
            float *gam = nullptr, *th = nullptr;
            const size_t b = (size_t)L * ctx->g.pitch * sizeof(float);
            if ((e = cudaMallocAsync((void**)&gam, b, s)) != cudaSuccess ||
                (e = cudaMallocAsync((void**)&th, b, s)) != cudaSuccess) {
                st = cuda_fail(e);
                break;
            }
            ctx->edge_gam[i - 1] = gam;
            ctx->edge_theta[i - 1] = th;
            ctx->edge_L[i - 1] = (int)L;
            st = run_launch(ctx, F_COEF, (double)H * ctx->g.W * 8.0, s, [&] {
                return launch_edge_profiles(ctx->dy, ctx->g, (int)L, ctx->kc[i - 1], gam, th, s);
            });
        }
    }
    if (st == DTS_OK && !comm && batch == 1 && ctx->A1y && opts_g().col_strips.load()) st = plan_strips(ctx, s);
    if (gstage) {
        cudaFreeAsync(gstage, s);
        if (st == DTS_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess) st = cuda_fail(e);
    }
    if (st != DTS_OK) {
        dts_destroy(ctx);
        return st;
    }
    ctx->last_stream = s;
    *out_ctx = ctx;
    return DTS_OK;
}

dts_status dts_create(const float* guide, int64_t H, int64_t W, int32_t C, float sigma_s, float sigma_r,
                      int32_t filter_passes, void* stream, dts_ctx** out_ctx) {
    return create_impl(guide, H, 0, H, W, C, sigma_s, sigma_r, filter_passes, nullptr, stream, out_ctx);
}

dts_status dts_create_batch(const float* guides, int64_t B, int64_t H, int64_t W, int32_t C, float sigma_s,
                            float sigma_r, int32_t filter_passes, void* stream, dts_ctx** out_ctx) {
    if (out_ctx) *out_ctx = nullptr;
    if (B < 1 || H < 1 || B > ((int64_t)1 << 30) / H) return B < 1 || H < 1 ? DTS_E_ARG : DTS_E_SHAPE;
    return create_impl(guides, B * H, 0, B * H, W, C, sigma_s, sigma_r, filter_passes, nullptr, stream, out_ctx, B);
}

// batched contexts: the FILTER column plan over the images as row strips (one launch holds every
// image's column tiles; HS = image height; no seam fix-up, the links between images are cut)
static bool batch_strip_plan(dts_ctx* ctx, int Ct, ColPlan* out) {
    if (ctx->batch < 2 || !ctx->A1y || Ct < 1 || Ct > 4 || opts_g().col_kernel.load() != 0) return false;
    if (ctx->bs_state[Ct] == 0) {
        Geometry gs = ctx->g;  // planned as the images side by side
        gs.H = ctx->batch_H;
        gs.W = ctx->g.W * ctx->batch;
        gs.pitch = (gs.W + 31) / 32 * 32;
        gs.plane = gs.H * gs.pitch;
        ColPlan ps{};
        const bool ok = gs.W <= ((int64_t)1 << 31) / 2 &&
                        plan_col(gs, Ct, MODE_FILTER, ctx->num_sms, &ps, opts_g().strip_cluster.load()) ==
                            cudaSuccess &&
                        ps.kind == 1 &&
                        colc_strips_supported(Ct, ps.Ls);
        cudaGetLastError();
        if (ok) {
            ps.HS = (int)ctx->batch_H;
            ps.ntc = (int)((ctx->g.W + 31) / 32);
            ps.ntiles = ps.ntc * (int)ctx->batch;
            ctx->bs_plan[Ct] = ps;
        }
        ctx->bs_state[Ct] = ok ? 1 : -1;
    }
    if (ctx->bs_state[Ct] != 1) return false;
    *out = ctx->bs_plan[Ct];
    return true;
}

// The FILTER column plan of a solve / confidence / stereo call for C_t: the batched strips, the
// create-time C_t = 1 strips, one cluster over the full height, or -- when no cluster holds
// the full height -- the fewest row strips whose columns fit one (a strip set built on first
// use: one stream sync), else the decoupled kernel.  *ss: the strip set whose seams need the
// fix-up (null for none).
static dts_status choose_col(dts_ctx* ctx, int Ct, cudaStream_t s, ColPlan* cp, StripSet** ss) {
    *ss = nullptr;
    if (batch_strip_plan(ctx, Ct, cp)) return DTS_OK;
    const bool strips_ok = !ctx->comm && ctx->batch == 1 && ctx->A1y && opts_g().col_strips.load() != 0 &&
                           opts_g().col_kernel.load() == 0;
    if (Ct == 1 && ctx->vs_set && strips_ok && strip_plan_n(ctx, ctx->vs_set->n, 1, cp)) {
        *ss = ctx->vs_set;
        return DTS_OK;
    }
    const cudaError_t e = ctx->comm ? plan_col_pass(ctx->g, Ct, MODE_FILTER, ctx->num_sms, cp)
                                    : plan_col(ctx->g, Ct, MODE_FILTER, ctx->num_sms, cp);
    cudaGetLastError();
    if (e == cudaSuccess && cp->kind == 1) return DTS_OK;
    if (strips_ok && Ct <= 3) {
        for (int n = 2; n <= 64; n *= 2) {
            ColPlan ps{};
            if (!strip_plan_n(ctx, n, Ct, &ps)) {
                if ((ctx->g.H + n - 1) / n < 64) break;
                continue;
            }
            StripSet* set = find_strip_set(ctx, n);
            if (!set) {
                const dts_status st = build_strip_set(ctx, n, s, &set);
                if (st != DTS_OK) return st;
                if (!set) break;  // the seam lengths do not fit: shorter strips would not either
            }
            *cp = ps;
            *ss = set;
            return DTS_OK;
        }
    }
    return e == cudaSuccess ? DTS_OK : DTS_E_SHAPE;
}

// Whether a FILTER column pass writes its output to the same planes of ctx->Xh instead of over
// its input in ctx->X (option col_oop; the next row pass then reads Xh and writes X).  Default 1:
// the passes over row strips, where the fused row update that follows the last one reads its
// z-bar input and writes its output in different buffers (C4: 466-468 against 476-481 us);
// 2: every cluster-kernel pass (no further gain on C4, C3 1.7% slower).
static bool col_oop(const dts_ctx* ctx, const ColPlan& cp, const StripSet* ss) {
    if (ctx->xh_failed) return false;
    const int o = opts_g().col_oop.load();
    return (o >= 1 && ss) || (o == 2 && cp.kind == 1 && ctx->A1y && ctx->N <= 4);
}

// where a FILTER column pass on (cp, ss) leaves the planes it read from ctx->X
static inline float* col_out(dts_ctx* ctx, const ColPlan& cp, const StripSet* ss) {
    return col_oop(ctx, cp, ss) ? ctx->Xh : ctx->X;
}

// the output planes of out-of-place column passes (ctx->Xh, as many planes as ctx->X)
static dts_status ensure_xh(dts_ctx* ctx, const ColPlan& cp, const StripSet* ss, cudaStream_t s) {
    if (!col_oop(ctx, cp, ss) || (ctx->Xh && ctx->xh_cap >= ctx->ct_cap)) return DTS_OK;
    if (ctx->Xh) cudaFreeAsync(ctx->Xh, s);
    ctx->Xh = nullptr;
    if (cudaMallocAsync((void**)&ctx->Xh, (size_t)ctx->g.plane * sizeof(float) * ctx->ct_cap, s) != cudaSuccess) {
        // an optimisation only: without the memory the passes run in place (same results)
        cudaGetLastError();
        ctx->Xh = nullptr;
        ctx->xh_failed = true;
        return DTS_OK;
    }
    ctx->xh_cap = ctx->ct_cap;
    return DTS_OK;
}

// FILTER column pass i over the C_t planes at x (x lies in ctx->X), on plan cp (choose_col): over
// row strips (ss) + the seam fix-up, the cluster kernel on A1 (image-high strips in batched
// contexts: cp.HS > 0), else the decoupled kernel on d_y.  The output lands at
// col_out(ctx, cp, ss) + (x - ctx->X).
static dts_status col_filter_pass(dts_ctx* ctx, const ColPlan& cp, const StripSet* ss, int Ct, int i, float* x,
                                  double bytes, cudaStream_t s) {
    const Geometry& g = ctx->g;
    float* xo = col_out(ctx, cp, ss) + (x - ctx->X);
    dts_status st = run_launch(ctx, F_COL, bytes, s, [&] {
        if (ss)  // row strips; the seams are fixed by the launch that follows
            return launch_col_cluster(cp, g, Ct, MODE_FILTER, x, ctx->A1y, ctx->kc[i], nullptr, nullptr, s, i,
                                      nullptr, nullptr, nullptr, ss->edge, xo);
        if (cp.kind == 1 && ctx->A1y && i < 4)
            return launch_col_cluster(cp, g, Ct, MODE_FILTER, x, ctx->A1y, ctx->kc[i], nullptr, nullptr, s, i,
                                      nullptr, nullptr, nullptr, nullptr, xo);
        return col_launch(ctx, cp, Ct, MODE_FILTER, x, ctx->dy, ctx->kc[i], nullptr, nullptr, s);
    });
    if (st == DTS_OK && ss)
        st = run_launch(ctx, F_SEAM, (double)g.W * 12.0 * Ct * (ss->n - 1) * 2 * ss->L[i], s, [&] {
            return launch_seam_fix(xo, Ct, g, ss->HS, ss->n, ss->L[i], ss->gam[i], ss->theta[i], ss->edge, s);
        });
    return st;
}

// debug hook (not in include/dts.h): the FILTER column plan dts_solve uses for C_t on this
// context -- out[0..6] = kind, CB, grid, threads, HS (0: one strip), ntiles, rows per segment
int32_t dts_debug_col_plan(dts_ctx* ctx, int32_t Ct, int32_t* out) {
    if (!ctx || !out || Ct < 1) return -1;
    ColPlan p{};
    StripSet* ss = nullptr;
    if (choose_col(ctx, Ct, ctx->last_stream, &p, &ss) != DTS_OK) return -1;
    const int32_t v[7] = {p.kind, p.CB, (int32_t)p.grid.x, p.threads, p.HS, p.ntiles, p.Ls};
    for (int i = 0; i < 7; ++i) out[i] = v[i];
    return 0;
}

// Box-filter context (reading R25): fixed-point increments, windows of every pass and the
// support, all computed once here.
static dts_status create_box_impl(const float* guide, int64_t H, int64_t W, int32_t C, float sigma_s, float sigma_r,
                                  int32_t filter_passes, double radius_scale, void* stream, dts_ctx** out_ctx) {
    if (!out_ctx || !guide) return DTS_E_ARG;
    *out_ctx = nullptr;
    if (H < 1 || W < 1 || C < 1) return DTS_E_ARG;
    if (!finite_pos(sigma_s) || !finite_pos(sigma_r)) return DTS_E_ARG;
    if (!(radius_scale >= 0.0) || !std::isfinite(radius_scale)) return DTS_E_ARG;
    if (filter_passes < 1 || filter_passes > 16) return DTS_E_ARG;
    if (W > ((int64_t)1 << 24) || H > ((int64_t)1 << 30) || C > 4096) return DTS_E_SHAPE;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int device = 0;
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(e);
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major < 10) {
        g_last_error = "device is not sm_100-class";
        return DTS_E_CUDA;
    }
    dts_ctx* ctx = new dts_ctx();
    ctx->filter = DTS_FILTER_BOX;
    ctx->device = device;
    ctx->H_total = H;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    ctx->g.H = H;
    ctx->g.W = W;
    ctx->g.pitch = (W + 31) / 32 * 32;
    ctx->g.plane = H * ctx->g.pitch;
    ctx->C = C;
    ctx->sigma_s = sigma_s;
    ctx->sigma_r = sigma_r;
    ctx->N = filter_passes;
    // radii in fixed point, R = floor(radius_scale * sigma * 2^16), sigma_i of R5 (the same
    // double expressions as the oracle's O2 / O10)
    std::vector<long long> R;
    const double denom = std::sqrt(std::pow(4.0, (double)filter_passes) - 1.0);
    for (int i = 1; i <= filter_passes; ++i) {
        const double sig = (double)sigma_s * std::sqrt(3.0) * std::pow(2.0, (double)(filter_passes - i)) / denom;
        R.push_back((long long)std::floor(radius_scale * sig * 65536.0));
    }
    R.push_back((long long)std::floor(radius_scale * (double)sigma_s * 65536.0));
    for (long long r : R)
        if ((r >> 16) > 65535) {  // window offsets are stored as 16-bit
            delete ctx;
            g_last_error = "box radius above 65535 pixels";
            return DTS_E_SHAPE;
        }
    for (int i = 0; i < filter_passes; ++i) {
        BoxPlan bp;
        if (plan_box(ctx->g, R[i], ctx->num_sms, &bp) != cudaSuccess) {
            cudaGetLastError();
            delete ctx;
            g_last_error = "box radius too large for the column tile";
            return DTS_E_SHAPE;
        }
        ctx->bplan.push_back(bp);
    }
    const PtrKind gk = classify(guide, device);
    if (gk == PTR_BAD) {
        delete ctx;
        return DTS_E_ARG;
    }
    const size_t plane = (size_t)ctx->g.plane * sizeof(float);
    dts_status st = DTS_OK;
    if ((e = cudaMallocAsync((void**)&ctx->dx_base, plane, s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->dy_base, plane, s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->S, plane, s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->win, plane * 2 * filter_passes, s)) != cudaSuccess ||
        (e = cudaMallocAsync((void**)&ctx->counters, 2 * sizeof(unsigned int), s)) != cudaSuccess) {
        st = cuda_fail(e);
        dts_destroy(ctx);
        return st;
    }
    ctx->dx = ctx->dx_base;
    ctx->dy = ctx->dy_base;
    const float* gdev = guide;
    float* gstage = nullptr;
    const size_t gbytes = (size_t)H * W * C * sizeof(float);
    if (gk == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&gstage, gbytes, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(gstage, guide, gbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
            st = cuda_fail(e);
            if (gstage) cudaFreeAsync(gstage, s);
            dts_destroy(ctx);
            return st;
        }
        gdev = gstage;
    }
    const float ratio = sigma_s / sigma_r;  // R25: k2 in fp32, as the oracle forms it
    const float k2 = ratio * ratio;
    uint32_t* qx = reinterpret_cast<uint32_t*>(ctx->dx);
    uint32_t* qy = reinterpret_cast<uint32_t*>(ctx->dy);
    const double px = (double)H * W;
    st = run_launch(ctx, F_BOX_PREP, px * (4.0 * C + 8.0), s,
                    [&] { return launch_box_increments(gdev, C, k2, ctx->g, qx, qy, s); });
    if (st == DTS_OK)
        st = run_launch(ctx, F_BOX_PREP, px * (8.0 + 8.0 * filter_passes + 4.0), s, [&] {
            return launch_box_windows(qx, qy, ctx->g, R.data(), (int)R.size(), ctx->win, ctx->S, s);
        });
    if (gstage) {
        cudaFreeAsync(gstage, s);
        if (st == DTS_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess) st = cuda_fail(e);
    }
    if (st != DTS_OK) {
        dts_destroy(ctx);
        return st;
    }
    ctx->last_stream = s;
    *out_ctx = ctx;
    return DTS_OK;
}

dts_status dts_create_ex(const float* guide, int64_t H, int64_t W, int32_t C, float sigma_s, float sigma_r,
                         int32_t filter_passes, const dts_create_opts* opts, void* stream, dts_ctx** out_ctx) {
    const int filter = opts ? opts->filter : DTS_FILTER_RF;
    if (filter == DTS_FILTER_RF)
        return create_impl(guide, H, 0, H, W, C, sigma_s, sigma_r, filter_passes, nullptr, stream, out_ctx);
    if (filter != DTS_FILTER_BOX) return DTS_E_ARG;
    if (opts->radius_scale < 0.f) return DTS_E_ARG;
    const double rs = (opts->radius_scale == 0.f) ? std::sqrt(3.0) : (double)opts->radius_scale;
    return create_box_impl(guide, H, W, C, sigma_s, sigma_r, filter_passes, rs, stream, out_ctx);
}

dts_status dts_debug_read_windows(dts_ctx* ctx, int32_t pass, int32_t axis, uint32_t* host_out) {
    if (!ctx || !host_out || ctx->filter != DTS_FILTER_BOX) return DTS_E_ARG;
    if (pass < 0 || pass >= ctx->N || (axis != 0 && axis != 1)) return DTS_E_ARG;
    const uint32_t* src = ctx->win + (size_t)(2 * pass + axis) * ctx->g.plane;
    cudaError_t e = cudaMemcpy2DAsync(host_out, ctx->g.W * sizeof(uint32_t), src, ctx->g.pitch * sizeof(uint32_t),
                                      ctx->g.W * sizeof(uint32_t), ctx->g.H, cudaMemcpyDeviceToHost, ctx->last_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->last_stream);
    return e == cudaSuccess ? DTS_OK : cuda_fail(e);
}

dts_status dts_create_band(const float* guide_with_halo, int64_t H_total, int64_t row0, int64_t rows, int64_t W,
                           int32_t C, float sigma_s, float sigma_r, int32_t filter_passes, dts_comm* comm,
                           void* stream, dts_ctx** out_ctx) {
    if (!comm) return create_impl(guide_with_halo, H_total, row0, rows, W, C, sigma_s, sigma_r, filter_passes,
                                  nullptr, stream, out_ctx);
    return create_impl(guide_with_halo, H_total, row0, rows, W, C, sigma_s, sigma_r, filter_passes, comm->c, stream,
                       out_ctx);
}

dts_status dts_comm_unique_id(void* id128) {
    if (!id128) return DTS_E_ARG;
    std::string err;
    if (!dts::nccl_unique_id(id128, &err)) {
        g_last_error = err;
        return DTS_E_NCCL;
    }
    return DTS_OK;
}

dts_status dts_comm_init(const void* id128, int32_t rank, int32_t nranks, dts_comm** out) {
    if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks || nranks > 64) return DTS_E_ARG;
    *out = nullptr;
    std::string err;
    dts::Comm* c = dts::comm_nccl(id128, rank, nranks, &err);
    if (!c) {
        g_last_error = err;
        return DTS_E_NCCL;
    }
    *out = new dts_comm{c};
    return DTS_OK;
}

dts_status dts_comm_init_loopback(int32_t nranks, dts_comm** comms) {
    if (!comms || nranks < 1 || nranks > 64) return DTS_E_ARG;
    std::vector<dts::Comm*> v = dts::comm_loopback(nranks);
    for (int r = 0; r < nranks; ++r) comms[r] = new dts_comm{v[r]};
    return DTS_OK;
}

void dts_comm_destroy(dts_comm* comm) {
    if (!comm) return;
    dts::comm_destroy(comm->c);
    delete comm;
}

dts_status dts_solve_ex(dts_ctx* ctx, const float* target, int32_t Ct, const float* confidence, float lambda,
                        int32_t iterations, float* out, void* stream, const dts_solve_opts* opts) {
    if (!ctx || !target || !confidence || !out) return DTS_E_ARG;
    if (Ct < 1) return DTS_E_ARG;
    if (Ct > 4) return DTS_E_SHAPE;
    if (iterations < 0) return DTS_E_ARG;
    const float step = (opts && opts->step > 0.f) ? opts->step : 0.99f;
    const int support_mode = opts ? opts->support_mode : 0;
    float* resid_out = opts ? opts->resid_inf_out : nullptr;
    if (support_mode != 0 && support_mode != 1) return DTS_E_ARG;
    if (!std::isfinite(lambda) || lambda < 0.f || !std::isfinite(step)) return DTS_E_ARG;
    if (step * (lambda + 1.f) >= 2.f) return DTS_E_ARG;  // descent stability
    const Geometry& g = ctx->g;
    const size_t img = (size_t)g.H * g.W * Ct * sizeof(float);
    const size_t cb = (size_t)g.H * g.W * sizeof(float);
    if (overlaps(out, img, target, img) || overlaps(out, img, confidence, cb)) return DTS_E_ARG;
    if (resid_out && (overlaps(resid_out, (size_t)iterations * 4, out, img) ||
                      overlaps(resid_out, (size_t)iterations * 4, target, img)))
        return DTS_E_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->last_stream = s;
    if (ctx->pend.on) {  // a solve that failed mid-way left an exchange pending: order after it
        ctx->pend.on = false;
        cudaStreamWaitEvent(s, ctx->ev_gath, 0);
    }

    const bool is_box = ctx->filter == DTS_FILTER_BOX;
    const bool want_resid = resid_out && iterations > 0;
    RowPlan rp{};
    ColPlan cpf{}, cpu{};
    StripSet* ssf = nullptr;  // row strips of the FILTER column passes (choose_col)
    int halves = 1;           // C_t = 4 without a cluster plan: two C_t = 2 halves
    if (!is_box) {
        if (plan_row_pass(g, Ct, MODE_FILTER, ctx->num_sms, &rp) != cudaSuccess && ctx->hs.n < 2) return DTS_E_SHAPE;
        cudaGetLastError();
        dts_status cs = choose_col(ctx, Ct, s, &cpf, &ssf);
        if (cs != DTS_OK) return cs;
        if (Ct == 4 && cpf.kind != 1 && !ctx->comm) {  // the cluster kernel has no C_t = 4 instance
            ColPlan c2{};
            StripSet* s2 = nullptr;
            if (choose_col(ctx, 2, s, &c2, &s2) == DTS_OK && c2.kind == 1) {
                cpf = c2;
                ssf = s2;
                halves = 2;
            }
        }
        // C_t >= 2 columns that need row strips run plane by plane: the one-plane strips use more
        // SMs (10000 x 10000 x 3: 97.8 against 107.3 ms per 20 iterations; 6000 x 4000 x 3 24.4
        // against 25.3), while columns one cluster holds stay joint (2160 x 3840 x 3: 8.0 against
        // 10.1 plane by plane).  Option col_split: 1 always plane by plane, 2 never.
        const int split = opts_g().col_split.load();
        if (Ct >= 2 && !ctx->comm && split != 2 && (split == 1 || ssf || cpf.kind != 1)) {
            ColPlan c1{};
            StripSet* s1 = nullptr;
            if (choose_col(ctx, 1, s, &c1, &s1) == DTS_OK && c1.kind == 1) {
                cpf = c1;
                ssf = s1;
                halves = Ct;
            }
        }
        // the decoupled kernel (tall columns) applies Eq. (3) in its own write-out
        if (cpf.kind != 1 && plan_col_pass(g, Ct, MODE_UPDATE, ctx->num_sms, &cpu) != cudaSuccess)
            return DTS_E_SHAPE;
        cudaGetLastError();
    }
    const PtrKind kt = classify(target, ctx->device), kc = classify(confidence, ctx->device),
                  ko = classify(out, ctx->device), kr = want_resid ? classify(resid_out, ctx->device) : PTR_DEVICE;
    if (kt == PTR_BAD || kc == PTR_BAD || ko == PTR_BAD || kr == PTR_BAD) return DTS_E_ARG;
    const bool any_host = kt == PTR_HOST || kc == PTR_HOST || ko == PTR_HOST || kr == PTR_HOST;
    cudaError_t e;
    dts_status st;
    if (any_host && (st = ensure_staging(ctx, img, s)) != DTS_OK) return st;
    const float* t_d = target;
    const float* c_d = confidence;
    float* o_d = out;
    if (kt == PTR_HOST) {
        if ((e = cudaMemcpyAsync(ctx->st_t, target, img, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e);
        t_d = ctx->st_t;
    }
    if (kc == PTR_HOST) {
        if ((e = cudaMemcpyAsync(ctx->st_c, confidence, cb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e);
        c_d = ctx->st_c;
    }
    if (ko == PTR_HOST) o_d = ctx->st_o;

    if (opts && opts->check_inputs) {
        unsigned int h[2] = {0, 0};
        if ((e = cudaMemsetAsync(ctx->counters, 0, sizeof(h), s)) != cudaSuccess) return cuda_fail(e);
        if ((e = launch_check_inputs(t_d, c_d, Ct, g.H, g.W, ctx->counters, s)) != cudaSuccess) return cuda_fail(e);
        ++ctx->launches;
        if ((e = cudaMemcpyAsync(h, ctx->counters, sizeof(h), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaStreamSynchronize(s)) != cudaSuccess)
            return cuda_fail(e);
        if (h[0]) return DTS_E_NONFINITE;
        if (h[1]) return DTS_E_RANGE;
    }
    // K8: per-iteration ||g||_inf, folded in by the update kernels (atomicMax of float bits)
    if (want_resid) {
        if (ctx->resid_cap < iterations) {
            if (ctx->resid) cudaFreeAsync(ctx->resid, s);
            ctx->resid = nullptr;
            ctx->resid_cap = 0;
            if ((e = cudaMallocAsync((void**)&ctx->resid, (size_t)iterations * sizeof(unsigned), s)) != cudaSuccess)
                return cuda_fail(e);
            ctx->resid_cap = iterations;
        }
        if ((e = cudaMemsetAsync(ctx->resid, 0, (size_t)iterations * sizeof(unsigned), s)) != cudaSuccess)
            return cuda_fail(e);
    }
    unsigned* resid = want_resid ? ctx->resid : nullptr;

    if (iterations == 0) {
        if ((e = cudaMemcpyAsync(o_d, t_d, img, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return cuda_fail(e);
    } else {
        if ((st = ensure_solver_state(ctx, Ct, s)) != DTS_OK) return st;
        if ((st = ensure_col_scratch(ctx, cpf, s)) != DTS_OK) return st;
        if ((st = ensure_col_scratch(ctx, cpu, s)) != DTS_OK) return st;
        if ((st = ensure_xh(ctx, cpf, ssf, s)) != DTS_OK) return st;
        auto enqueue = [&](cudaStream_t s) -> dts_status {
            dts_status st;
            const double px = (double)g.H * g.W;
            st = run_launch(ctx, F_PROLOGUE, px * (12.0 * Ct + 12 + (ctx->Sy ? 4.0 : 0.0)), s, [&] {
                return launch_prologue(t_d, c_d, Ct, g, ctx->S, ctx->Sy, support_mode, ctx->Z, ctx->T, ctx->chat, s);
            });
            if (st != DTS_OK) return st;
            const double row_bytes = px * (8.0 * Ct + 4);
            const double upd_bytes = px * (16.0 * Ct + 8);  // X, d, Z, T, chat in; Z out
            if (is_box) {  // R25: N x (box rows, box columns), ping-pong X2 <-> X, then Eq. (3)
                for (int k = 0; k < iterations; ++k) {
                    for (int i = 0; i < ctx->N; ++i) {
                        const BoxPlan& bp = ctx->bplan[i];
                        const uint32_t* wx = ctx->win + (size_t)(2 * i) * g.plane;
                        const uint32_t* wy = ctx->win + (size_t)(2 * i + 1) * g.plane;
                        const float* in = (i == 0) ? ctx->Z : ctx->X;
                        st = run_launch(ctx, F_BOX_ROW, row_bytes, s,
                                        [&] { return launch_box_row(bp, g, Ct, in, ctx->X2, wx, s); });
                        if (st != DTS_OK) return st;
                        st = run_launch(ctx, F_BOX_COL, row_bytes, s,
                                        [&] { return launch_box_col(bp, g, Ct, ctx->X2, ctx->X, wy, s); });
                        if (st != DTS_OK) return st;
                    }
                    float* ohwc = (k + 1 == iterations) ? o_d : nullptr;
                    st = run_launch(ctx, F_STEP, px * (16.0 * Ct + 4), s, [&] {
                        return launch_update(ctx->X, ctx->Z, ctx->T, ctx->chat, Ct, g, lambda, step, ohwc,
                                             ctx->num_sms, s, resid ? resid + k : nullptr);
                    });
                    if (st != DTS_OK) return st;
                }
                return DTS_OK;
            }
            // The last column pass of an iteration is a FILTER pass; Eq. (3) of iteration k-1 is
            // applied inside iteration k's first row pass (k_row.cu ROWUPD: Z, T, chat read
            // coalesced while the row lands) and one update kernel closes the solve.  The
            // decoupled kernel (tall columns) applies Eq. (3) in its own write-out instead; with
            // the residual requested the step runs as its own kernel every iteration.
            const bool split_update = cpf.kind == 1 || ctx->comm || want_resid;
            const bool rowupd = split_update && !want_resid && opts_g().row_update.load();
            UpdateArgs ru;
            ru.Z = ctx->Z;
            ru.T = ctx->T;
            ru.chat = ctx->chat;
            ru.lam = lambda;
            ru.step = step;
            ru.out_hwc = nullptr;
            ru.resid = nullptr;
            // row pass i over rows [r0, r0 + n) (the whole band, or part of it around a pending
            // edge fix-up); upd: Eq. (3) of the previous iteration applied on the fly
            auto row_rows = [&](int i, const float* in, bool upd, int64_t r0, int64_t n) -> dts_status {
                if (upd)
                    return row_pass_x(ctx, Ct, MODE_FILTER, i, in, ctx->X, &ru, r0, n, F_ROWUPD,
                                      (double)n * g.W * (20.0 * Ct + 8), s);
                return row_pass_x(ctx, Ct, MODE_FILTER, i, in, ctx->X, nullptr, r0, n, F_ROW,
                                  (double)n * g.W * (8.0 * Ct + 4), s);
            };
            float* xc = ctx->X;  // the planes the last column pass wrote (col_out)
            for (int k = 0; k < iterations; ++k) {
                for (int i = 0; i < ctx->N; ++i) {
                    const bool upd = rowupd && i == 0 && k > 0;  // Eq. (3) of iteration k-1 in this row pass
                    const float* in = (i == 0 && !upd) ? ctx->Z : xc;
                    if (ctx->pend.on) {
                        // overlapped band exchange: interior rows while the all-gather runs, then
                        // the edge fix-up and the 2L edge rows
                        const int64_t L = std::min<int64_t>(ctx->pend.L, g.H / 2);
                        st = row_rows(i, in, upd, L, g.H - 2 * L);
                        if (st == DTS_OK) st = finish_pending(ctx, s);
                        if (st == DTS_OK) st = row_rows(i, in, upd, 0, L);
                        if (st == DTS_OK) st = row_rows(i, in, upd, g.H - L, L);
                    } else {
                        st = row_rows(i, in, upd, 0, g.H);
                    }
                    if (st != DTS_OK) return st;
                    const bool last = i + 1 == ctx->N;
                    float* ohwc = (k + 1 == iterations) ? o_d : nullptr;
                    if (ctx->comm) {  // row-band mode: the exchange of DESIGN.md section 9
                        if (!last || (rowupd && k + 1 < iterations)) {  // a row pass follows: overlap
                            st = col_pass_banded(ctx, Ct, MODE_FILTER, ctx->X, ctx->kc[i], nullptr, nullptr, F_COL,
                                                 row_bytes, s, i, opts_g().band_overlap.load() != 0);
                        } else {
                            UpdateArgs u = ru;
                            u.out_hwc = ohwc;
                            u.resid = resid ? resid + k : nullptr;
                            st = col_pass_banded(ctx, Ct, MODE_UPDATE, ctx->X, ctx->kc[i], &u, nullptr, F_UPDATE,
                                                 upd_bytes, s, i);
                        }
                    } else if (!last || split_update) {
                        for (int h = 0; h < halves && st == DTS_OK; ++h)
                            st = col_filter_pass(ctx, cpf, ssf, Ct / halves, i, ctx->X + h * (Ct / halves) * g.plane,
                                                 row_bytes / halves, s);
                        if (st != DTS_OK) return st;
                        xc = col_out(ctx, cpf, ssf);
                        if (!last || (rowupd && k + 1 < iterations)) continue;  // the next row pass applies Eq. (3)
                        st = run_launch(ctx, F_STEP, px * (16.0 * Ct + 4), s, [&] {
                            return launch_update(xc, ctx->Z, ctx->T, ctx->chat, Ct, g, lambda, step, ohwc,
                                                 ctx->num_sms, s, resid ? resid + k : nullptr);
                        });
                    } else {  // decoupled kernel: Eq. (3) in the column write-out
                        UpdateArgs u = ru;
                        u.out_hwc = ohwc;
                        st = run_launch(ctx, F_UPDATE, upd_bytes, s, [&] {
                            return col_launch(ctx, cpu, Ct, MODE_UPDATE, ctx->X, ctx->dy, ctx->kc[i], &u, nullptr, s);
                        });
                    }
                    if (st != DTS_OK) return st;
                }
            }
            return DTS_OK;
        };
        // Replay a captured graph of the whole launch sequence when the same solve is issued
        // again (small images are launch-bound).  Only on the cluster column path or the box
        // path (no per-launch epochs), with device buffers and the profiler off.
        const bool use_graph = opts_g().graphs.load() && !any_host && !profiler_on() && !ctx->comm &&
                               (is_box || cpf.kind == 1);
        std::vector<uintptr_t> key;
        if (use_graph) {
            uint32_t lb, sb;
            std::memcpy(&lb, &lambda, 4);
            std::memcpy(&sb, &step, 4);
            key = {1, (uintptr_t)t_d, (uintptr_t)c_d, (uintptr_t)o_d, (uintptr_t)Ct, (uintptr_t)iterations, lb, sb,
                   (uintptr_t)support_mode, (uintptr_t)ctx->X, (uintptr_t)ctx->Xh, (uintptr_t)ctx->Z, (uintptr_t)ctx->chat,
                   (uintptr_t)resid};
        }
        if ((st = run_cached(ctx, use_graph, key, s, enqueue)) != DTS_OK) return st;
    }
    if (ko == PTR_HOST) {
        if ((e = cudaMemcpyAsync(out, o_d, img, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return cuda_fail(e);
    }
    if (want_resid &&
        (e = cudaMemcpyAsync(resid_out, ctx->resid, (size_t)iterations * sizeof(float), cudaMemcpyDefault, s)) !=
            cudaSuccess)
        return cuda_fail(e);
    if (any_host) {
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e);
    }
    return DTS_OK;
}

dts_status dts_confidence(dts_ctx* ctx, const float* target, float sigma_c, float* conf_out, float* var_out,
                          void* stream) {
    if (ctx && ctx->filter != DTS_FILTER_RF) return DTS_E_ARG;  // recursive-filter contexts only
    if (!ctx || !target || !conf_out) return DTS_E_ARG;
    if (!std::isfinite(sigma_c) || !(sigma_c > 0.f)) return DTS_E_ARG;
    if (ctx->comm) return DTS_E_SHAPE;  // row-band contexts: not supported (yet)
    const Geometry& g = ctx->g;
    const size_t cb = (size_t)g.H * g.W * sizeof(float);
    if (overlaps(conf_out, cb, target, cb) || (var_out && (overlaps(var_out, cb, target, cb) ||
                                                           overlaps(var_out, cb, conf_out, cb))))
        return DTS_E_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->last_stream = s;
    RowPlan rp;
    ColPlan cp{}, cp1{};
    if (plan_row_pass(g, 2, MODE_FILTER, ctx->num_sms, &rp) != cudaSuccess && ctx->hs.n < 2) return DTS_E_SHAPE;
    cudaGetLastError();
    StripSet *ss2 = nullptr, *ss1 = nullptr;
    const bool two = choose_col(ctx, 2, s, &cp, &ss2) == DTS_OK;
    // when two planes do not fit the cluster column kernel (tall images) but one does, or one
    // plane's plan covers >= 10% more SMs (C4: C_t = 1 strips on 135 SMs against C_t = 2 strips
    // on 112: 2.9 against 3.3 ms per call), the column passes run plane by plane
    const bool one = choose_col(ctx, 1, s, &cp1, &ss1) == DTS_OK && cp1.kind == 1;
    const bool per_plane = one && (!(two && cp.kind == 1) || cp1.grid.x * 10 >= cp.grid.x * 11);
    cudaGetLastError();
    if (!two && !per_plane) return DTS_E_SHAPE;
    const PtrKind kt = classify(target, ctx->device), kc = classify(conf_out, ctx->device),
                  kv = var_out ? classify(var_out, ctx->device) : PTR_DEVICE;
    if (kt == PTR_BAD || kc == PTR_BAD || kv == PTR_BAD) return DTS_E_ARG;
    const bool any_host = kt == PTR_HOST || kc == PTR_HOST || kv == PTR_HOST;
    dts_status st;
    cudaError_t e;
    if (any_host && (st = ensure_staging(ctx, cb, s)) != DTS_OK) return st;
    const float* t_d = target;
    float* c_d = kc == PTR_HOST ? ctx->st_o : conf_out;
    float* v_d = (var_out && kv == PTR_HOST) ? ctx->st_c : var_out;
    if (kt == PTR_HOST) {
        if ((e = cudaMemcpyAsync(ctx->st_t, target, cb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e);
        t_d = ctx->st_t;
    }
    if ((st = ensure_solver_state(ctx, 2, s)) != DTS_OK) return st;
    if (!per_plane && (st = ensure_col_scratch(ctx, cp, s)) != DTS_OK) return st;
    const double px = (double)g.H * g.W;
    // planes [t ; t^2] -> DTF (N passes of rows then columns) -> Eq. (7)
    if ((st = (per_plane ? ensure_xh(ctx, cp1, ss1, s) : ensure_xh(ctx, cp, ss2, s))) != DTS_OK) return st;
    st = run_launch(ctx, F_CONF, px * 12.0, s, [&] { return launch_conf_prologue(t_d, g, ctx->X, s); });
    float* xc = ctx->X;  // the planes the last column pass wrote (col_out)
    for (int i = 0; i < ctx->N && st == DTS_OK; ++i) {
        st = row_pass_x(ctx, 2, MODE_FILTER, i, xc, ctx->X, nullptr, 0, g.H, F_ROW, px * 20.0, s);
        if (st == DTS_OK && !per_plane) st = col_filter_pass(ctx, cp, ss2, 2, i, ctx->X, px * 20.0, s);
        for (int v = 0; v < 2 && st == DTS_OK && per_plane; ++v)
            st = col_filter_pass(ctx, cp1, ss1, 1, i, ctx->X + v * g.plane, px * 12.0, s);
        xc = per_plane ? col_out(ctx, cp1, ss1) : col_out(ctx, cp, ss2);
    }
    const float inv = 1.f / (2.f * sigma_c * sigma_c);
    if (st == DTS_OK)
        st = run_launch(ctx, F_CONF, px * (var_out ? 16.0 : 12.0), s,
                        [&] { return launch_conf_epilogue(xc, g, inv, c_d, v_d, s); });
    if (st != DTS_OK) return st;
    if (kc == PTR_HOST && (e = cudaMemcpyAsync(conf_out, c_d, cb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e);
    if (var_out && kv == PTR_HOST && (e = cudaMemcpyAsync(var_out, v_d, cb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e);
    if (any_host && (e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e);
    return DTS_OK;
}

dts_status dts_solve_stereo(dts_ctx* ctx, const float* target, const float* confidence, float lambda,
                            int32_t iterations, float* out, const float* left, const float* right, float gamma,
                            float eps, void* stream) {
    if (ctx && ctx->filter != DTS_FILTER_RF) return DTS_E_ARG;  // recursive-filter contexts only
    if (!ctx || !target || !confidence || !out || !left || !right) return DTS_E_ARG;
    if (iterations < 0) return DTS_E_ARG;
    const float step = 0.99f;
    if (!std::isfinite(lambda) || lambda < 0.f || step * (lambda + 1.f) >= 2.f) return DTS_E_ARG;
    if (!std::isfinite(gamma) || gamma < 0.f || !std::isfinite(eps) || !(eps > 0.f)) return DTS_E_ARG;
    if (ctx->comm) return DTS_E_SHAPE;  // row-band contexts: not supported (yet)
    const Geometry& g = ctx->g;
    const size_t cb = (size_t)g.H * g.W * sizeof(float);
    const size_t gb = cb * (size_t)ctx->C;
    if (overlaps(out, cb, target, cb) || overlaps(out, cb, confidence, cb) || overlaps(out, cb, left, gb) ||
        overlaps(out, cb, right, gb))
        return DTS_E_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->last_stream = s;
    RowPlan rp;
    ColPlan cp{};
    StripSet* ss1 = nullptr;
    if (plan_row_pass(g, 1, MODE_FILTER, ctx->num_sms, &rp) != cudaSuccess && ctx->hs.n < 2) return DTS_E_SHAPE;
    if (choose_col(ctx, 1, s, &cp, &ss1) != DTS_OK) return DTS_E_SHAPE;
    cudaGetLastError();
    const PtrKind kt = classify(target, ctx->device), kc = classify(confidence, ctx->device),
                  ko = classify(out, ctx->device), kl = classify(left, ctx->device), kr = classify(right, ctx->device);
    if (kt == PTR_BAD || kc == PTR_BAD || ko == PTR_BAD || kl == PTR_BAD || kr == PTR_BAD) return DTS_E_ARG;
    const bool any_host = kt == PTR_HOST || kc == PTR_HOST || ko == PTR_HOST || kl == PTR_HOST || kr == PTR_HOST;
    dts_status st = DTS_OK;
    cudaError_t e;
    if (any_host && (st = ensure_staging(ctx, cb, s)) != DTS_OK) return st;
    const float* t_d = target;
    const float* c_d = confidence;
    float* o_d = ko == PTR_HOST ? ctx->st_o : out;
    float *l_tmp = nullptr, *r_tmp = nullptr;
    const float* l_d = left;
    const float* r_d = right;
    auto cleanup = [&]() {
        if (l_tmp) cudaFreeAsync(l_tmp, s);
        if (r_tmp) cudaFreeAsync(r_tmp, s);
    };
    if (kt == PTR_HOST) {
        if ((e = cudaMemcpyAsync(ctx->st_t, target, cb, cudaMemcpyHostToDevice, s)) != cudaSuccess) return cuda_fail(e);
        t_d = ctx->st_t;
    }
    if (kc == PTR_HOST) {
        if ((e = cudaMemcpyAsync(ctx->st_c, confidence, cb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e);
        c_d = ctx->st_c;
    }
    if (kl == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&l_tmp, gb, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(l_tmp, left, gb, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
            cleanup();
            return cuda_fail(e);
        }
        l_d = l_tmp;
    }
    if (kr == PTR_HOST) {
        if ((e = cudaMallocAsync((void**)&r_tmp, gb, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(r_tmp, right, gb, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
            cleanup();
            return cuda_fail(e);
        }
        r_d = r_tmp;
    }
    if (iterations == 0) {
        if ((e = cudaMemcpyAsync(o_d, t_d, cb, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) st = cuda_fail(e);
    } else {
        if (st == DTS_OK) st = ensure_solver_state(ctx, 1, s);
        if (st == DTS_OK) st = ensure_col_scratch(ctx, cp, s);
        if (st == DTS_OK) st = ensure_xh(ctx, cp, ss1, s);
        const double px = (double)g.H * g.W;
        auto enqueue = [&](cudaStream_t s) -> dts_status {
            dts_status st = run_launch(ctx, F_PROLOGUE, px * (24.0 + (ctx->Sy ? 4.0 : 0.0)), s, [&] {
                return launch_prologue(t_d, c_d, 1, g, ctx->S, ctx->Sy, 0, ctx->Z, ctx->T, ctx->chat, s);
            });
            float* xc = ctx->X;  // the planes the last column pass wrote (col_out)
            for (int k = 0; k < iterations && st == DTS_OK; ++k) {
                for (int i = 0; i < ctx->N && st == DTS_OK; ++i) {
                    const float* in = (i == 0) ? ctx->Z : xc;
                    st = row_pass_x(ctx, 1, MODE_FILTER, i, in, ctx->X, nullptr, 0, g.H, F_ROW, px * 12.0, s);
                    if (st == DTS_OK) st = col_filter_pass(ctx, cp, ss1, 1, i, ctx->X, px * 12.0, s);
                    xc = col_out(ctx, cp, ss1);
                }
                float* ohw = (k + 1 == iterations) ? o_d : nullptr;
                if (st == DTS_OK)
                    st = run_launch(ctx, F_STEREO, px * (20.0 + 12.0 * ctx->C), s, [&] {
                        return launch_update_stereo(xc, ctx->Z, ctx->T, ctx->chat, l_d, r_d, ctx->C, g, lambda,
                                                    step, gamma, eps, ohw, s);
                    });
            }
            return st;
        };
        if (st == DTS_OK) {
            const bool use_graph = opts_g().graphs.load() && !any_host && !profiler_on() && cp.kind == 1;
            std::vector<uintptr_t> key;
            if (use_graph) {
                uint32_t lb, gb2, eb;
                std::memcpy(&lb, &lambda, 4);
                std::memcpy(&gb2, &gamma, 4);
                std::memcpy(&eb, &eps, 4);
                key = {2, (uintptr_t)t_d, (uintptr_t)c_d, (uintptr_t)o_d, (uintptr_t)l_d, (uintptr_t)r_d,
                       (uintptr_t)iterations, lb, gb2, eb, (uintptr_t)ctx->X, (uintptr_t)ctx->Xh, (uintptr_t)ctx->Z,
                       (uintptr_t)ctx->chat};
            }
            st = run_cached(ctx, use_graph, key, s, enqueue);
        }
    }
    if (st == DTS_OK && ko == PTR_HOST &&
        (e = cudaMemcpyAsync(out, o_d, cb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        st = cuda_fail(e);
    cleanup();
    if (st == DTS_OK && any_host && (e = cudaStreamSynchronize(s)) != cudaSuccess) st = cuda_fail(e);
    return st;
}

dts_status dts_solve(dts_ctx* ctx, const float* target, int32_t target_channels, const float* confidence,
                     float lambda, int32_t iterations, float* out, void* stream) {
    return dts_solve_ex(ctx, target, target_channels, confidence, lambda, iterations, out, stream, nullptr);
}

void dts_destroy(dts_ctx* ctx) {
    if (!ctx) return;
    cudaStream_t s = ctx->last_stream;
    free_solver_state(ctx, s);
    ctx->A1y = nullptr;
    for (float** p : {&ctx->dx_base, &ctx->dy_base, &ctx->S, &ctx->Sy, &ctx->A1y_base, &ctx->st_t, &ctx->st_c, &ctx->st_o,
                      &ctx->rank_tup, &ctx->gathered, &ctx->ext}) {
        if (*p) cudaFreeAsync(*p, s);
        *p = nullptr;
    }
    if (ctx->counters) cudaFreeAsync(ctx->counters, s);
    if (ctx->tuples) cudaFreeAsync(ctx->tuples, s);
    if (ctx->flags) cudaFreeAsync(ctx->flags, s);
    if (ctx->resid) cudaFreeAsync(ctx->resid, s);
    if (ctx->win) cudaFreeAsync(ctx->win, s);
    for (float* q : ctx->edge_gam)
        if (q) cudaFreeAsync(q, s);
    for (float* q : ctx->edge_theta)
        if (q) cudaFreeAsync(q, s);
    for (StripSet* ss : ctx->ssets) {
        for (float* q : ss->gam)
            if (q) cudaFreeAsync(q, s);
        for (float* q : ss->theta)
            if (q) cudaFreeAsync(q, s);
        if (ss->edge) cudaFreeAsync(ss->edge, s);
        delete ss;
    }
    for (float* q : ctx->hs_gam)
        if (q) cudaFreeAsync(q, s);
    for (float* q : ctx->hs_theta)
        if (q) cudaFreeAsync(q, s);
    if (ctx->graph_exec) {  // a replay may still be in flight on s
        cudaStreamSynchronize(s);
        cudaGraphExecDestroy(ctx->graph_exec);
    }
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->comm_stream) {
        cudaStreamSynchronize(ctx->comm_stream);
        cudaStreamDestroy(ctx->comm_stream);
    }
    if (ctx->ev_cols) cudaEventDestroy(ctx->ev_cols);
    if (ctx->ev_gath) cudaEventDestroy(ctx->ev_gath);
    delete ctx;
}

dts_status dts_debug_read(dts_ctx* ctx, dts_buffer which, float* host_out) {
    if (!ctx || !host_out) return DTS_E_ARG;
    const float* src = which == DTS_BUF_DX ? ctx->dx : which == DTS_BUF_DY ? ctx->dy
                     : which == DTS_BUF_SUPPORT ? ctx->S : nullptr;
    if (!src) return DTS_E_ARG;
    cudaError_t e = cudaMemcpy2DAsync(host_out, ctx->g.W * sizeof(float), src, ctx->g.pitch * sizeof(float),
                                      ctx->g.W * sizeof(float), ctx->g.H, cudaMemcpyDeviceToHost, ctx->last_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->last_stream);
    if (e == cudaSuccess && which == DTS_BUF_SUPPORT && ctx->Sy) {  // S = s_x * s_y
        std::vector<float> sy((size_t)ctx->g.H * ctx->g.W);
        e = cudaMemcpy2DAsync(sy.data(), ctx->g.W * sizeof(float), ctx->Sy, ctx->g.pitch * sizeof(float),
                              ctx->g.W * sizeof(float), ctx->g.H, cudaMemcpyDeviceToHost, ctx->last_stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->last_stream);
        if (e == cudaSuccess)
            for (size_t i = 0; i < sy.size(); ++i) host_out[i] *= sy[i];
    }
    return e == cudaSuccess ? DTS_OK : cuda_fail(e);
}

dts_status dts_profile_enable(dts_ctx* ctx, int32_t on) {
    (void)ctx;  // the profiler is process-wide
    Profiler& P = profiler();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e);
    std::lock_guard<std::mutex> lk(P.mu);
    P.resolve();
    for (auto& f : P.fam) {  // (re)starting resets the statistics
        f.launches = 0;
        f.total_ms = 0;
    }
    P.on = on != 0;
    return DTS_OK;
}

dts_status dts_profile_read(dts_ctx* ctx, dts_kernel_stat* out, int32_t max, int32_t* count) {
    (void)ctx;
    Profiler& P = profiler();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e);
    std::lock_guard<std::mutex> lk(P.mu);
    P.resolve();
    int n = 0;
    for (auto& f : P.fam) {
        if (out && n < max) {
            std::memset(&out[n], 0, sizeof(dts_kernel_stat));
            std::strncpy(out[n].name, f.name.c_str(), sizeof(out[n].name) - 1);
            out[n].launches = f.launches;
            out[n].total_ms = f.total_ms;
            out[n].bytes_per_launch = f.bytes_per_launch;
        }
        ++n;
    }
    if (count) *count = n;
    return DTS_OK;
}

int64_t dts_launch_count(const dts_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
