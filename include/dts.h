/*
 * dts.h -- C ABI of the B200-native Domain Transform Solver hot path.
 *
 * The method: Bapat & Frahm, "The Domain Transform Solver" (arXiv 1805.04590).
 * Citations: P:n = /root/reference/PAPER.md line n; "R<k>" = reading k in
 * DESIGN.md "Readings of the paper".
 *
 * The library solves, for a guide image I and a target t with confidence c,
 *     min_z  lambda/2 sum_i (z_i - zbar_i)^2 + sum_i c_i (z_i - t_i)^2        (Eq. 2)
 * by the gradient descent of P:481 / P:567:
 *     z <- z - step * [ lambda (z - zbar) + (c / S) (z - t) ]                  (Eq. 3)
 * where zbar = DTF(z) is the edge-aware mean computed with the domain
 * transform as N passes of Gastal & Oliveira's recursive filter
 * along rows then columns (R3-R6), and S = sum_j W_ij is the filter's support
 * (R7).
 *
 * Conventions shared by every entry point:
 *  - Images are fp32, C-contiguous, row-major, channel-interleaved (HWC):
 *    element (r, c, k) of an H x W x C image is at [(r * W + c) * C + k].
 *  - Array arguments may be CUDA DEVICE pointers or HOST pointers (pageable or
 *    page-locked); the library tells them apart with cudaPointerGetAttributes.
 *    Host arrays are copied to/from device staging buffers owned by the context
 *    on `stream`; when any argument of a call is host memory the call returns
 *    only after its results are in host memory (it synchronises `stream`).
 *    With device pointers every call is asynchronous and stream-ordered.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *  - Ownership: the caller owns every array it passes; the library never frees
 *    or retains a caller pointer after the call returns.  A dts_ctx owns its
 *    derived buffers (domain distances, support, solver state) until
 *    dts_destroy.  One context must not be used from two streams at once;
 *    distinct contexts are independent.
 *  - Errors: every entry point validates its scalar arguments on the host
 *    before any launch and returns a dts_status; on error nothing is launched
 *    and the outputs are untouched.  DTS_E_CUDA reports a CUDA launch/runtime
 *    error (dts_last_error_string gives the CUDA message).  There is NO CPU
 *    fallback: if the CUDA runtime or an sm_100a device is missing, calls fail.
 *  - Results are deterministic: identical inputs on the same device give
 *    bit-identical outputs (no atomics on the data path).
 */
#ifndef DTS_B200_H
#define DTS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dts_ctx dts_ctx; /* opaque; owned by the library */

typedef enum {
    DTS_OK = 0,
    DTS_E_ARG = 1,       /* invalid scalar argument or NULL / overlapping pointer      */
    DTS_E_SHAPE = 2,     /* sizes outside what this build supports (see dts_create)   */
    DTS_E_NONFINITE = 3, /* non-finite input detected (opt-in checks)                  */
    DTS_E_RANGE = 4,     /* confidence outside [0, 1] (opt-in checks)                  */
    DTS_E_CUDA = 5,      /* CUDA runtime / launch error, or no sm_100 device           */
    DTS_E_NCCL = 6,      /* collective error (row-band mode)                           */
    DTS_E_OOM = 7        /* device or host allocation failed                           */
} dts_status;

/* dts_create -- domain-transform setup for one guide image.
 *   guide          H x W x C fp32, HWC; read once.  Colours are used as given (no
 *                  clamping, R16); only differences of adjacent pixels matter.
 *   H, W, C        >= 1.  W <= 184320: the row kernel stages whole rows of every plane in
 *                  shared memory (11520 columns at C_t = 4); wider rows run over up to 16
 *                  vertical strips with a seam fix-up, which needs
 *                  every pass's carry-decay length L (measured at create) to fit twice in a
 *                  strip -- else DTS_E_SHAPE.  Columns taller than one thread-block
 *                  cluster holds (10240 rows at C_t = 1, 7168 at 2, 5632 at 3) run over row
 *                  strips with a seam fix-up (the first dts_solve that needs them measures
 *                  the strips' seam lengths: one sync of its stream), else -- a seam length
 *                  longer than half a strip, N > 4 -- over the decoupled kernel, which
 *                  bounds H per context: on a 148-SM B200 at least 30000 rows for C_t = 1
 *                  and 6400 for C_t = 3.  A larger H returns DTS_E_SHAPE (from dts_create,
 *                  or from dts_solve for the C_t of that call); split such images into row
 *                  bands (dts_create_band).
 *   sigma_s        spatial std-dev in pixels (sigma_x = sigma_y), > 0, finite.
 *   sigma_r        range std-dev in colour units, > 0, finite.
 *   filter_passes  N >= 1 recursive-filter passes per edge-aware mean (R5); N <= 16.
 * Computes the horizontal / vertical domain distances
 *     d = sqrt(1 + (sigma_s/sigma_r)^2 * sum_k (I_k(p) - I_k(p'))^2)      (Eqs. 8-9, R1, R2)
 * with +inf at the first column / row, and the support S = s_x * s_y (R7).
 * On success *out_ctx receives a new context (release with dts_destroy).    */
dts_status dts_create(const float* guide, int64_t H, int64_t W, int32_t C,
                      float sigma_s, float sigma_r, int32_t filter_passes,
                      void* stream, dts_ctx** out_ctx);

/* dts_create_batch -- one context for B independent images of the same size (the C3
 * workload, "eight 4K images"; north star "independent images ... per rank").
 *   guides         B x H x W x C fp32 (B HWC images back to back); read once.
 *   B, H, W, C     B >= 1, B * H <= 2^30; otherwise as dts_create.
 * The context is the B images stacked into one (B*H) x W image whose column recurrences
 * are cut between consecutive images (d_y = +inf at each image's first row: the
 * first-row rule R4 of every image), so every call on it -- dts_solve / dts_solve_ex with
 * target and confidence B x H x W [x C_t], dts_confidence, dts_debug_read -- treats the
 * images exactly as B separate contexts would (the recurrence restarts are exact: the cut
 * coefficient is 0).  What batching buys: each column pass launches every image's column
 * tiles at once (a per-C_t plan over image-high strips), every row pass all B*H rows.
 * The per-context row limit above applies to the image height H (C_t <= 3 with the A1
 * coefficient, N <= 4); other configurations fall back to the stacked-image plans and the
 * (B*H)-row limits.  Errors: as dts_create; DTS_E_SHAPE when B * H > 2^30.          */
dts_status dts_create_batch(const float* guides, int64_t B, int64_t H, int64_t W, int32_t C,
                            float sigma_s, float sigma_r, int32_t filter_passes,
                            void* stream, dts_ctx** out_ctx);

/* dts_solve -- `iterations` gradient-descent steps of Eq. (3) with
 * step 0.99, starting from z^0 = t (R11).
 *   target            H x W x target_channels fp32, HWC.  Channels are solved
 *                     independently with the same filter (R14).
 *   target_channels   C_t >= 1 (this build: 1 <= C_t <= 4).
 *   confidence        H x W fp32, one channel shared by all target channels, c >= 0
 *                     (values are not range-checked unless dts_solve_ex asks).
 *   lambda            smoothness weight, finite, >= 0, and step*(lambda + 1) < 2
 *                     (descent stability); the paper uses 0.99.
 *   iterations        >= 0; 0 copies target to out exactly.
 *   out               H x W x C_t fp32, HWC; must not overlap target or confidence.
 * Each iteration recomputes zbar = DTF(z) (R12) and applies
 *     z <- z - 0.99 * [ lambda (z - zbar) + (c / S) (z - t) ].                  */
dts_status dts_solve(dts_ctx* ctx, const float* target, int32_t target_channels,
                     const float* confidence, float lambda, int32_t iterations,
                     float* out, void* stream);

/* dts_destroy -- releases the context and its device buffers.  NULL-safe.  */
void dts_destroy(dts_ctx* ctx);

/* Human-readable name of a status code (static storage). */
const char* dts_status_string(dts_status s);

/* Message of the last CUDA error seen by this thread (static storage, "" if none). */
const char* dts_last_error_string(void);

/* ---- extensions used by the tests and the benchmark -------------------- */

typedef struct {
    float step;          /* gradient step; <= 0 selects the paper's 0.99        */
    int32_t support_mode;/* 0: S = s_x * s_y (R7, default); 1: S = 1 (unweighted c)     */
    int32_t check_inputs;/* 1: verify finite target/confidence and c in [0,1] (syncs)   */
    float* resid_inf_out;/* NULL, or `iterations` floats (device or host memory): entry k
                            receives ||g_k||_inf, the max-norm of the Eq. (3) gradient
                            g_k = lambda (z^k - zbar^k) + chat (z^k - t) at iterate k
                            (reading R13), over all pixels and channels of this
                            context (row-band contexts: of this rank's rows).  Computed on
                            the device inside the update kernels (a max: deterministic).
                            Must not overlap `out` or `target`.                            */
} dts_solve_opts;

/* dts_solve with options; opts == NULL is exactly dts_solve. */
dts_status dts_solve_ex(dts_ctx* ctx, const float* target, int32_t target_channels,
                        const float* confidence, float lambda, int32_t iterations,
                        float* out, void* stream, const dts_solve_opts* opts);

/* ---- box (normalised-convolution) variant of the edge-aware mean ---------
 * P:243-245 write the mean with the box indicator W_ij = delta{DT(z_i) - DT(z_j) <= r};
 * reading R25 takes it as the normalised window on the guide's
 * domain-transform axis, zbar_i = (1/|N_i|) sum_{j in N_i} z_j, N_i = {j : |T_j - T_i| <= r},
 * N passes of rows then columns with r_i = radius_scale * sigma_i (R5 schedule), and the
 * support S = |N^x| * |N^y| at r = radius_scale * sigma_s.  Window
 * membership is exact integer arithmetic: d is evaluated in IEEE fp32 in a fixed order
 * (k2 = (sigma_s/sigma_r)^2 in fp32, s = sum_k dI_k^2 in channel order, d = sqrt(1 + k2 s),
 * no fused multiply-add) and T is held in fixed point, q = round_half_even(d * 2^16) capped
 * at 2^30, R = floor(r * 2^16) (double). */
typedef enum { DTS_FILTER_RF = 0, DTS_FILTER_BOX = 1 } dts_filter;
typedef struct {
    int32_t filter;      /* DTS_FILTER_RF (default, what dts_create builds) or DTS_FILTER_BOX  */
    float radius_scale;  /* box: r_i = radius_scale * sigma_i; 0 selects sqrt(3), < 0 is
                            DTS_E_ARG.  Ignored for DTS_FILTER_RF                               */
} dts_create_opts;

/* dts_create with options; opts == NULL (or filter == DTS_FILTER_RF) is exactly dts_create.
 * A box context supports dts_solve / dts_solve_ex (same arguments and semantics, with the
 * box mean and the box support in Eq. 3); dts_confidence and dts_solve_stereo return
 * DTS_E_ARG for it.  Box limits: window half-width <= 65535 px, and the column tile needs
 * min(floor(r_1), H - 1) <= ~800 rows (else DTS_E_SHAPE).  Memory: 2N window planes
 * (4 B/px each) + the fixed-point increments (8 B/px) + S, plus a second state buffer
 * per solve. */
dts_status dts_create_ex(const float* guide, int64_t H, int64_t W, int32_t C, float sigma_s, float sigma_r,
                         int32_t filter_passes, const dts_create_opts* opts, void* stream, dts_ctx** out_ctx);

/* Box context only: copy the windows of pass `pass` (0-based) along `axis` (0: rows,
 * 1: columns) to host_out (H x W uint32, row-major): lo | hi << 16, the window of pixel
 * i along the line being [i - lo, i + hi].  Synchronises the context's last stream. */
dts_status dts_debug_read_windows(dts_ctx* ctx, int32_t pass, int32_t axis, uint32_t* host_out);

/* Confidence from the edge-aware variance, Eq. (7) of the paper:
 *     V_i = DT(t_i^2) - DT(t_i)^2   (clamped at 0),     c_i = exp(-V_i / (2 sigma_c^2))
 * where DT is the context's N-pass edge-aware mean (the same recursive filter and
 * coefficients dts_solve uses) and t a one-channel target, e.g. the disparity
 * whose confidence feeds dts_solve.  SURVEY 8(f) #1.
 *   target     H x W fp32 (device or host pointer), finite.
 *   sigma_c    variance scale, finite, > 0 (the paper gives no value; SPEC S:210 uses 16
 *              disparity units as a default).
 *   conf_out   H x W fp32, receives c in (0, 1]; must not overlap target.
 *   var_out    optional (NULL allowed) H x W fp32, receives V >= 0.
 * Stream-ordered like dts_solve; host pointers are staged (and the call synchronises).
 * Errors: DTS_E_ARG (NULL / overlapping pointers, sigma_c <= 0 or not finite),
 *         DTS_E_CUDA / DTS_E_OOM from the device.  Uses the context's solver buffers,
 *         so it must not run concurrently with dts_solve on the same context. */
dts_status dts_confidence(dts_ctx* ctx, const float* target, float sigma_c, float* conf_out, float* var_out,
                          void* stream);

/* Stereo refinement, Eq. (10) of the paper: gradient descent on
 *     lambda/2 sum (z - zbar)^2 + sum c rho(z - t) + 1/2 sum gamma ||I_L(i) - I_R(i - z_i)||^2
 * with the Charbonnier rho(r) = sqrt(r^2 + eps^2) on the target term (the paper uses
 * eps = 0.001, gamma = 0.001).  Each iteration: the context's N-pass
 * edge-aware mean zbar, then z <- z - step [lambda (z - zbar) + chat rho'(z - t)
 * + gamma sum_k (I_L,k(x) - I_R,k(x - z)) dI_R,k/dx(x - z)], chat = c / S (R7), I_R sampled
 * by linear interpolation along the row (rectified pair), clamped, slope 0 outside the
 * image (reading R23).  z^0 = t.  SURVEY 8(f) #2.
 *   target, confidence, out  H x W fp32 (one channel: the disparity), as dts_solve.
 *   left, right  H x W x C fp32 HWC, C = the context's guide channels; `left` is the
 *                image the context was created from, `right` its stereo partner.
 *   gamma        photometric weight, finite, >= 0 (0: only the robust target term).
 *   eps          Charbonnier epsilon, finite, > 0.
 * Pointers may be host or device (host arrays are staged; the call then synchronises).
 * Errors: DTS_E_ARG (NULL / overlapping pointers, bad scalars as in dts_solve),
 *         DTS_E_SHAPE (row-band contexts), DTS_E_CUDA / DTS_E_OOM. */
dts_status dts_solve_stereo(dts_ctx* ctx, const float* target, const float* confidence, float lambda,
                            int32_t iterations, float* out, const float* left, const float* right, float gamma,
                            float eps, void* stream);

/* Depth super-resolution front end: from an h x w low-resolution
 * depth map, the target and confidence of an (h f) x (w f) DTS solve (use them with a context
 * built on the high-resolution colour guide):
 *   target = bicubic upsampling ("simple bicubic interpolation"): Catmull-Rom kernel
 *            (a = -0.5), separable, clamped borders, centre-aligned (low-res sample k at
 *            high-res coordinate k f + (f - 1)/2);
 *   conf   = Gaussian bump around the nearest low-res sample centre:
 *            exp(-dist^2 / (2 sigma_b^2)), sigma_b = f / 4 (reading R24).
 *   low            h x w fp32 (device or host); target_out, conf_out (h f) x (w f) fp32.
 *   factor         integer >= 1 (f = 1 copies `low` and sets conf = 1).
 * Context-free; stream-ordered (host pointers are staged and the call synchronises).
 * Errors: DTS_E_ARG (NULL pointers, h, w or factor < 1, outputs overlapping `low` or each
 *         other), DTS_E_CUDA / DTS_E_OOM. */
dts_status dts_sr_prepare(const float* low, int64_t h, int64_t w, int32_t factor, float* target_out,
                          float* conf_out, void* stream);

/* Buffers a test can read back (row-major H x W, fp32; stream-ordered then synchronised). */
typedef enum { DTS_BUF_DX = 0, DTS_BUF_DY = 1, DTS_BUF_SUPPORT = 2 } dts_buffer;
/* Copies the H x W buffer `which` into host memory `host_out` (H*W floats).  Box
 * contexts: DX / DY hold the fixed-point increments q as uint32 bit patterns (view the
 * floats as uint32), SUPPORT the window-count product. */
dts_status dts_debug_read(dts_ctx* ctx, dts_buffer which, float* host_out);

/* Per-kernel timing with CUDA events recorded on the launch stream around every
 * launch of the library's kernels (off by default; costs one event pair per launch).
 * The profiler is PROCESS-WIDE (statistics survive dts_destroy, so a timed step may
 * create and destroy contexts); `ctx` is ignored and may be NULL.  Both calls
 * synchronise the device.  Enabling (or re-enabling) resets the statistics. */
typedef struct {
    char name[32];          /* kernel family: deriv, row_pass, col_pass, col_update, ...  */
    int64_t launches;       /* launches timed since dts_profile_enable                    */
    double total_ms;        /* sum of event-measured durations                            */
    double bytes_per_launch;/* algorithmic HBM bytes of one launch            */
} dts_kernel_stat;
dts_status dts_profile_enable(dts_ctx* ctx, int32_t on);
/* Fills up to `max` records; *count receives the number of kernel families. */
dts_status dts_profile_read(dts_ctx* ctx, dts_kernel_stat* out, int32_t max, int32_t* count);

/* Number of kernel launches issued by the library since context creation (all streams). */
int64_t dts_launch_count(const dts_ctx* ctx);

/* ---- row-band mode: one tall image split across processes / GPUs -------- */
/* Rows [row0, row0 + rows) of an H_total x W image live on one rank.  Row passes stay
 * local; every column pass exchanges one 5-tuple per column per rank (an all-gather of
 * (2 C_t + 3) x W floats) and composes the carries into the rank's rows (DESIGN.md
 * "Multi-GPU"; reading R20).  Results equal the single-context solve to fp32 rounding. */
typedef struct dts_comm dts_comm; /* opaque; owned by the library */

/* 128-byte NCCL unique id for dts_comm_init (call on one rank, broadcast the bytes). */
dts_status dts_comm_unique_id(void* id128);
/* NCCL communicator over `nranks` processes; rank r owns the r-th band in row order.
 * The calling thread's current CUDA device is used.  NCCL is loaded at run time
 * (libnccl.so.2 already in the process, else $DTS_NCCL_LIB); failures -> DTS_E_NCCL. */
dts_status dts_comm_init(const void* id128, int32_t rank, int32_t nranks, dts_comm** out);
/* `nranks` communicators for ranks that are host THREADS of this process sharing one
 * GPU (testing the row-band algebra without several GPUs): comms[r] for r < nranks.
 * Each thread drives its own context on its own stream; collective calls rendezvous
 * on the host. */
dts_status dts_comm_init_loopback(int32_t nranks, dts_comm** comms);
void dts_comm_destroy(dts_comm* comm); /* NULL-safe; destroy after the contexts using it */

/* dts_create_band -- like dts_create for rows [row0, row0 + rows) of an H_total-row image.
 *   guide_with_halo  (rows + above + below) x W x C, HWC: the band's guide rows preceded
 *                    by the row above (above = 1 if row0 > 0, else 0) and followed by the
 *                    row below (below = 1 if row0 + rows < H_total) -- needed for the
 *                    vertical domain distances at the seams (R20).
 *   comm             communicator whose ranks own consecutive bands in rank order; NULL
 *                    only for a single band (row0 = 0, rows = H_total).
 * COLLECTIVE: every rank of `comm` calls dts_create_band (and later dts_solve, with the
 * same target_channels / lambda / iterations) with its own band.  dts_solve on a band
 * context takes and returns the band's rows (rows x W target / confidence / out). */
dts_status dts_create_band(const float* guide_with_halo, int64_t H_total, int64_t row0, int64_t rows,
                           int64_t W, int32_t C, float sigma_s, float sigma_r, int32_t filter_passes,
                           dts_comm* comm, void* stream, dts_ctx** out_ctx);

/* ---- test / experiment options (process-wide; the defaults are the product path) ----
 * dts_set_option(name, value) selects among equivalent implementations so that tests can
 * check each against the oracle; it never changes what is computed.  Names and values:
 *   "col_kernel"   0 cluster column kernel when a column tile fits a cluster (default),
 *                  1 the decoupled band-tuple kernel everywhere
 *   "band_scheme"  row-band contexts (latched at dts_create_band): 0 edge fix-up where the
 *                  bands allow it (default), 1 cluster TUPLE/APPLY, 2 decoupled kernel
 *   "band_overlap" row-band contexts, edge scheme: 1 (default) the all-gather of a column pass
 *                  runs on a context stream while the next row pass filters the band's
 *                  interior rows; 0 serial (same results, bit for bit)
 *   "col_split"    C_t >= 2 column passes: 0 (default) plane by plane when the columns need
 *                  row strips, 1 always plane by plane, 2 never
 *   "row_seg"      row-kernel samples per thread: 0 auto (default), 4, 12, 20, 36
 *   "pdl"          programmatic dependent launch of the hot-path kernels: 1 (default) with the
 *                  dependent launch triggered at the end of each kernel, 2 at the start, 0 off
 *   "graphs"       1 replay repeated identical solves as CUDA graphs (default), 0 never
 *   "row_update"   1 Eq. (3) step fused into the next iteration's first row pass (default)
 *   "col_rows"     0 auto (default); rows per warp segment of the cluster column kernel: 32 or
 *                  40 (C_t = 1), 12 or 16 (C_t = 3)
 *   "col_cluster"  0 auto (default), 1..16: forced column-kernel cluster size
 *   "col_strips"   tall single images: row strips for the C_t = 1 column passes, 0 off,
 *                  1 auto (default), n >= 2 exactly n strips when they fit
 *   "strip_cluster" 0 auto (default), 1..16: forced cluster size of a row-strip plan
 *   "col_oop"      column passes out of place into a second state buffer: 0 never, 1 the
 *                  passes over row strips (default), 2 every cluster-kernel pass
 *   "row_two_ctas" C_t = 3 row passes of <= 3840 columns: 1 two CTAs per SM (default), 0 one
 * Returns DTS_E_ARG for an unknown name or value.  dts_get_option returns -1 for unknown names. */
dts_status dts_set_option(const char* name, int32_t value);
int32_t dts_get_option(const char* name);

/* Library version string. */
const char* dts_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DTS_B200_H */
