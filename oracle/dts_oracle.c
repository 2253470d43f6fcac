/*
 * dts_oracle.c -- plain, slow, fp64 CPU oracle for the Domain Transform Solver
 * (Bapat & Frahm, "The Domain Transform Solver", arXiv 1805.04590).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_1805_04590_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * "Qk" = the reading numbered k in SURVEY.md 8(c), restated in DESIGN.md.
 *
 * Every routine below is the definition written out with plain loops in double
 * precision, in the paper's order and notation:
 *   O1 dts_oracle_distances   P:231-240 (Eqs. 8-9, square restored, Q1/Q2)
 *   O2 dts_oracle_sigmas      recursive-filter pass schedule (Q5)
 *   O3 dts_oracle_rf1d        recursive filter, causal then anticausal (Q4)
 *   O4 dts_oracle_dtf         2-D edge-aware mean: rows then columns, per pass (Q6)
 *   O5 dts_oracle_support     S = sum_j W_ij by unnormalised two-sided sums (Q7)
 *   O6 dts_oracle_solve       gradient descent on Eq. (2) with the Eq. (3) gradient
 *   O7 dts_oracle_confidence  Eq. (7) confidence from the edge-aware variance
 *   O8 dts_oracle_solve_stereo Eq. (10) stereo refinement with the Charbonnier target term
 *   O9 dts_oracle_sr_prepare  depth-SR front end
 *   O10 dts_oracle_box_*      box (normalised-convolution) edge-aware mean, its support and
 *                             the DTS iteration with it (reading R25)
 * Parallelism: OpenMP "parallel for" over independent rows / column ranges only;
 * each output element is produced by exactly one thread with the same
 * arithmetic, so results do not depend on the thread count.  Reductions for
 * diagnostics are serial.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_E_ARG 1
#define ORACLE_E_OOM 7

int dts_oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void dts_oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------------ */
/* O1: domain-transform increments between adjacent pixels.
 * (DT(x+h) - DT(x))^2 = h^2 + sum_k (I(x+h)-I(x))^2 (the L2 isometry,
 * P:231); with the spatial/range scales of the experiments
 * folded in as in S:125 (reading Q2):
 *     d_x[r][c] = sqrt(1 + (sigma_s/sigma_r)^2 * sum_k (I[r][c][k] - I[r][c-1][k])^2),  c >= 1
 *     d_x[r][0] = +inf   (no left neighbour: the recursion restarts, reading Q4)
 * and d_y the same along columns (d_y[0][c] = +inf).
 * guide: H x W x C fp32, HWC interleaved.  dx, dy: H x W doubles, row-major.  */
int dts_oracle_distances(const float* guide, int64_t H, int64_t W, int32_t C,
                         double sigma_s, double sigma_r, double* dx, double* dy) {
    if (!guide || !dx || !dy || H < 1 || W < 1 || C < 1) return ORACLE_E_ARG;
    if (!(sigma_s > 0.0) || !(sigma_r > 0.0)) return ORACLE_E_ARG;
    const double ratio = sigma_s / sigma_r;
    const double ratio2 = ratio * ratio;
    int64_t r;
#pragma omp parallel for schedule(static)
    for (r = 0; r < H; ++r) {
        for (int64_t c = 0; c < W; ++c) {
            /* horizontal neighbour (r, c-1) */
            if (c == 0) {
                dx[r * W + c] = INFINITY;
            } else {
                double sum = 0.0;
                for (int32_t k = 0; k < C; ++k) {
                    double diff = (double)guide[(r * W + c) * C + k] - (double)guide[(r * W + c - 1) * C + k];
                    sum += diff * diff;
                }
                dx[r * W + c] = sqrt(1.0 + ratio2 * sum);
            }
            /* vertical neighbour (r-1, c) */
            if (r == 0) {
                dy[r * W + c] = INFINITY;
            } else {
                double sum = 0.0;
                for (int32_t k = 0; k < C; ++k) {
                    double diff = (double)guide[(r * W + c) * C + k] - (double)guide[((r - 1) * W + c) * C + k];
                    sum += diff * diff;
                }
                dy[r * W + c] = sqrt(1.0 + ratio2 * sum);
            }
        }
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* O2: per-pass standard deviations of the N-pass recursive filter (reading Q5):
 *     sigma_i = sigma_s * sqrt(3) * 2^(N-i) / sqrt(4^N - 1),  i = 1..N
 * so that sum_i sigma_i^2 = sigma_s^2; the pass-i feedback is a_i = exp(-sqrt(2)/sigma_i)
 * and the per-pixel coefficient is a_i^d = exp(-sqrt(2) d / sigma_i). */
void dts_oracle_sigmas(double sigma_s, int32_t N, double* sigma_i) {
    const double denom = sqrt(pow(4.0, (double)N) - 1.0);
    for (int32_t i = 1; i <= N; ++i)
        sigma_i[i - 1] = sigma_s * sqrt(3.0) * pow(2.0, (double)(N - i)) / denom;
}

/* coefficient a^d for pass sigma: exp(-sqrt(2) * d / sigma); exp(-inf) = 0 */
static double rf_coef(double d, double sigma) {
    return exp(-sqrt(2.0) * d / sigma);
}

/* ------------------------------------------------------------------------ */
/* O3: one recursive-filter pass over a 1-D signal of n samples, spaced `stride`
 * elements apart (reading Q4; the recurrence is the one BASELINE.json's
 * north star restates, J[n] = (1 - a^d) I[n] + a^d J[n-1]):
 *     causal:      y[0] = x[0];        y[k] = (1 - A[k]) x[k] + A[k] y[k-1]
 *     anticausal:  z[n-1] = y[n-1];    z[k] = (1 - A[k+1]) y[k] + A[k+1] z[k+1]
 * A[0] is not used (the +inf sentinel makes it 0).  In place: x <- z. */
void dts_oracle_rf1d(double* x, const double* A, int64_t n, int64_t stride) {
    if (n <= 0) return;
    /* causal */
    for (int64_t k = 1; k < n; ++k) {
        double a = A[k * stride];
        x[k * stride] = (1.0 - a) * x[k * stride] + a * x[(k - 1) * stride];
    }
    /* anticausal */
    for (int64_t k = n - 2; k >= 0; --k) {
        double a = A[(k + 1) * stride];
        x[k * stride] = (1.0 - a) * x[k * stride] + a * x[(k + 1) * stride];
    }
}

/* ------------------------------------------------------------------------ */
/* O4: the 2-D edge-aware mean  zbar = DTF(z)  ("two passes, once in the
 * X direction and once in Y"; P:249 alternating X then Y; N passes with the O2
 * schedule, reading Q5/Q6).  For i = 1..N: every row is filtered with
 * A_i^x = exp(-sqrt2 d_x / sigma_i), then every column with A_i^y.
 * X: Ct planes of H x W doubles, filtered in place; channels are independent
 * (reading Q14).  Ax, Ay: per-pass coefficient arrays, N x H x W each.       */
static void dtf_with_coefs(double* X, int64_t H, int64_t W, int32_t Ct, int32_t N,
                           const double* Ax, const double* Ay) {
    for (int32_t i = 0; i < N; ++i) {
        const double* ax = Ax + (int64_t)i * H * W;
        const double* ay = Ay + (int64_t)i * H * W;
        for (int32_t ch = 0; ch < Ct; ++ch) {
            double* P = X + (int64_t)ch * H * W;
            /* rows: each row is one 1-D signal */
            int64_t r;
#pragma omp parallel for schedule(static)
            for (r = 0; r < H; ++r) dts_oracle_rf1d(P + r * W, ax + r * W, W, 1);
            /* columns, row-streaming: the same recurrence as dts_oracle_rf1d
             * along each column, evaluated for all columns of a range at once
             * so that memory is walked row by row. */
            const int64_t block = 256;
            const int64_t nblk = (W + block - 1) / block;
            int64_t b;
#pragma omp parallel for schedule(static)
            for (b = 0; b < nblk; ++b) {
                const int64_t c0 = b * block;
                const int64_t c1 = (c0 + block < W) ? c0 + block : W;
                for (int64_t k = 1; k < H; ++k)          /* causal, top -> bottom */
                    for (int64_t c = c0; c < c1; ++c) {
                        double a = ay[k * W + c];
                        P[k * W + c] = (1.0 - a) * P[k * W + c] + a * P[(k - 1) * W + c];
                    }
                for (int64_t k = H - 2; k >= 0; --k)     /* anticausal, bottom -> top */
                    for (int64_t c = c0; c < c1; ++c) {
                        double a = ay[(k + 1) * W + c];
                        P[k * W + c] = (1.0 - a) * P[k * W + c] + a * P[(k + 1) * W + c];
                    }
            }
        }
    }
}

static int make_coefs(const double* dx, const double* dy, int64_t H, int64_t W,
                      double sigma_s, int32_t N, double** Ax_out, double** Ay_out) {
    double sig[64];
    if (N < 1 || N > 64) return ORACLE_E_ARG;
    dts_oracle_sigmas(sigma_s, N, sig);
    double* Ax = (double*)malloc(sizeof(double) * (size_t)N * (size_t)H * (size_t)W);
    double* Ay = (double*)malloc(sizeof(double) * (size_t)N * (size_t)H * (size_t)W);
    if (!Ax || !Ay) { free(Ax); free(Ay); return ORACLE_E_OOM; }
    for (int32_t i = 0; i < N; ++i) {
        int64_t p;
#pragma omp parallel for schedule(static)
        for (p = 0; p < H * W; ++p) {
            Ax[(int64_t)i * H * W + p] = rf_coef(dx[p], sig[i]);
            Ay[(int64_t)i * H * W + p] = rf_coef(dy[p], sig[i]);
        }
    }
    *Ax_out = Ax;
    *Ay_out = Ay;
    return ORACLE_OK;
}

/* DTF of Ct planar channels given the O1 distances.  X (Ct x H x W) in place. */
int dts_oracle_dtf(double* X, int64_t H, int64_t W, int32_t Ct,
                   const double* dx, const double* dy, double sigma_s, int32_t N) {
    if (!X || !dx || !dy || H < 1 || W < 1 || Ct < 1 || N < 1) return ORACLE_E_ARG;
    double *Ax = NULL, *Ay = NULL;
    int st = make_coefs(dx, dy, H, W, sigma_s, N, &Ax, &Ay);
    if (st) return st;
    dtf_with_coefs(X, H, W, Ct, N, Ax, Ay);
    free(Ax);
    free(Ay);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* O5: support S_i = sum_j W_ij ("weigh the confidence c_i ... by
 * sum_j W_ij"), for the recursive-filter kernel (reading Q7): separable
 * unnormalised two-sided exponential sums with a = exp(-sqrt2 / sigma_s),
 *     P[k] = 1 + a^{d[k]} P[k-1],  P[0] = 1
 *     Q[k] = 1 + a^{d[k+1]} Q[k+1], Q[n-1] = 1
 *     s = P + Q - 1     (each pixel counts itself once: W_ii = 1)
 * along rows (s_x, with d_x) and along columns (s_y, with d_y); S = s_x * s_y.
 * support_mode 1 gives S = 1 (the unweighted A/B option of Q7).             */
int dts_oracle_support(const double* dx, const double* dy, int64_t H, int64_t W,
                       double sigma_s, int32_t support_mode, double* S) {
    if (!dx || !dy || !S || H < 1 || W < 1 || !(sigma_s > 0.0)) return ORACLE_E_ARG;
    if (support_mode == 1) {
        for (int64_t p = 0; p < H * W; ++p) S[p] = 1.0;
        return ORACLE_OK;
    }
    double* sx = (double*)malloc(sizeof(double) * (size_t)H * (size_t)W);
    double* P = (double*)malloc(sizeof(double) * (size_t)(H > W ? H : W));
    double* Q = (double*)malloc(sizeof(double) * (size_t)(H > W ? H : W));
    if (!sx || !P || !Q) { free(sx); free(P); free(Q); return ORACLE_E_OOM; }
    /* rows (serial: create-time, plain) */
    for (int64_t r = 0; r < H; ++r) {
        const double* d = dx + r * W;
        P[0] = 1.0;
        for (int64_t k = 1; k < W; ++k) P[k] = 1.0 + rf_coef(d[k], sigma_s) * P[k - 1];
        Q[W - 1] = 1.0;
        for (int64_t k = W - 2; k >= 0; --k) Q[k] = 1.0 + rf_coef(d[k + 1], sigma_s) * Q[k + 1];
        for (int64_t k = 0; k < W; ++k) sx[r * W + k] = P[k] + Q[k] - 1.0;
    }
    /* columns */
    for (int64_t c = 0; c < W; ++c) {
        P[0] = 1.0;
        for (int64_t k = 1; k < H; ++k) P[k] = 1.0 + rf_coef(dy[k * W + c], sigma_s) * P[k - 1];
        Q[H - 1] = 1.0;
        for (int64_t k = H - 2; k >= 0; --k) Q[k] = 1.0 + rf_coef(dy[(k + 1) * W + c], sigma_s) * Q[k + 1];
        for (int64_t k = 0; k < H; ++k) S[k * W + c] = sx[k * W + c] * (P[k] + Q[k] - 1.0);
    }
    free(sx);
    free(P);
    free(Q);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* O6: the DTS iteration (Eqs. 3-4; step 0.99):
 *     chat = c / S                                        (reading Q7)
 *     Z^0 = T                                             (reading Q11)
 *     for k = 0..iters-1:
 *         zbar = DTF(Z^k)                                  (recomputed every iteration, Q12)
 *         g    = lambda (Z^k - zbar) + chat (Z^k - T)      (Eq. 3 as printed, Q8)
 *         Z^{k+1} = Z^k - step * g
 * guide: H x W x Cg fp32 HWC; target: H x W x Ct fp32 HWC; confidence: H x W fp32
 * (one channel broadcast over Ct, Q14).  out: H x W x Ct doubles HWC.
 * diag (optional, iters x 4 doubles): per iteration k, computed at Z^k:
 *     [0] ||g||_inf   [1] ||g||_2
 *     [2] Fhat = lambda/2 ||Z - zbar||^2 + 1/2 sum chat (Z - T)^2
 *     [3] Eq  = lambda/2 Z.(Z - zbar) + 1/2 sum chat (Z - T)^2
 * (reading Q13: the residual norms are asserted monotone, the objectives only
 * reported).                                                                  */
int dts_oracle_solve(const float* guide, int64_t H, int64_t W, int32_t Cg,
                     double sigma_s, double sigma_r, int32_t N,
                     const float* target, int32_t Ct, const float* confidence,
                     double lambda, double step, int32_t iters, int32_t support_mode,
                     double* out, double* diag) {
    if (!guide || !target || !confidence || !out) return ORACLE_E_ARG;
    if (H < 1 || W < 1 || Cg < 1 || Ct < 1 || N < 1 || iters < 0) return ORACLE_E_ARG;
    const int64_t HW = H * W;
    double* dx = (double*)malloc(sizeof(double) * (size_t)HW);
    double* dy = (double*)malloc(sizeof(double) * (size_t)HW);
    double* S = (double*)malloc(sizeof(double) * (size_t)HW);
    double* chat = (double*)malloc(sizeof(double) * (size_t)HW);
    double* Z = (double*)malloc(sizeof(double) * (size_t)HW * (size_t)Ct);
    double* T = (double*)malloc(sizeof(double) * (size_t)HW * (size_t)Ct);
    double* Zbar = (double*)malloc(sizeof(double) * (size_t)HW * (size_t)Ct);
    double *Ax = NULL, *Ay = NULL;
    int st = ORACLE_OK;
    if (!dx || !dy || !S || !chat || !Z || !T || !Zbar) { st = ORACLE_E_OOM; goto done; }

    st = dts_oracle_distances(guide, H, W, Cg, sigma_s, sigma_r, dx, dy);        /* O1 */
    if (st) goto done;
    st = dts_oracle_support(dx, dy, H, W, sigma_s, support_mode, S);            /* O5 */
    if (st) goto done;
    st = make_coefs(dx, dy, H, W, sigma_s, N, &Ax, &Ay);                        /* O2 */
    if (st) goto done;

    for (int64_t p = 0; p < HW; ++p) chat[p] = (double)confidence[p] / S[p];
    /* planar copies of the target: channel ch of pixel p at [ch*HW + p] */
    for (int32_t ch = 0; ch < Ct; ++ch)
        for (int64_t p = 0; p < HW; ++p) {
            T[ch * HW + p] = (double)target[p * Ct + ch];
            Z[ch * HW + p] = T[ch * HW + p];
        }

    for (int32_t k = 0; k < iters; ++k) {
        memcpy(Zbar, Z, sizeof(double) * (size_t)HW * (size_t)Ct);
        dtf_with_coefs(Zbar, H, W, Ct, N, Ax, Ay);                              /* O4 */
        if (diag) {
            double ginf = 0.0, g2 = 0.0, fhat = 0.0, eq = 0.0;
            for (int32_t ch = 0; ch < Ct; ++ch)
                for (int64_t p = 0; p < HW; ++p) {
                    double z = Z[ch * HW + p], zb = Zbar[ch * HW + p], t = T[ch * HW + p];
                    double g = lambda * (z - zb) + chat[p] * (z - t);
                    if (fabs(g) > ginf) ginf = fabs(g);
                    g2 += g * g;
                    fhat += 0.5 * lambda * (z - zb) * (z - zb) + 0.5 * chat[p] * (z - t) * (z - t);
                    eq += 0.5 * lambda * z * (z - zb) + 0.5 * chat[p] * (z - t) * (z - t);
                }
            diag[4 * k + 0] = ginf;
            diag[4 * k + 1] = sqrt(g2);
            diag[4 * k + 2] = fhat;
            diag[4 * k + 3] = eq;
        }
        int64_t q;
#pragma omp parallel for schedule(static)
        for (q = 0; q < HW * Ct; ++q) {
            int64_t p = q % HW;
            double g = lambda * (Z[q] - Zbar[q]) + chat[p] * (Z[q] - T[q]);        /* Eq. (3) */
            Z[q] = Z[q] - step * g;
        }
    }
    for (int32_t ch = 0; ch < Ct; ++ch)
        for (int64_t p = 0; p < HW; ++p) out[p * Ct + ch] = Z[ch * HW + p];

done:
    free(dx); free(dy); free(S); free(chat); free(Z); free(T); free(Zbar);
    free(Ax); free(Ay);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O7: confidence from the edge-aware variance (Eq. 7):
 *     V_i = DT(z_i^2) - DT(z_i)^2,    c_i = exp(-V_i / (2 sigma_c^2))
 * "the domain transform is treated as a local estimate of the mean in an edge-aware
 * sense": DT is the O4 edge-aware mean DTF with the guide's coefficients, and
 * z is the target (the confidence of the MC-CNN disparity target).  V is
 * clamped at 0 (DTF is a convex combination, so V >= 0 up to rounding; reading R22).
 * target: H x W fp32 (one channel); conf, var (optional): H x W doubles.         */
int dts_oracle_confidence(const float* guide, int64_t H, int64_t W, int32_t Cg,
                          double sigma_s, double sigma_r, int32_t N,
                          const float* target, double sigma_c, double* conf, double* var) {
    if (!guide || !target || !conf || H < 1 || W < 1 || Cg < 1 || N < 1) return ORACLE_E_ARG;
    if (!(sigma_c > 0.0)) return ORACLE_E_ARG;
    const int64_t HW = H * W;
    double* dx = (double*)malloc(sizeof(double) * (size_t)HW);
    double* dy = (double*)malloc(sizeof(double) * (size_t)HW);
    double* X = (double*)malloc(sizeof(double) * (size_t)HW * 2);  /* [z ; z^2] planar */
    int st = ORACLE_OK;
    if (!dx || !dy || !X) { st = ORACLE_E_OOM; goto done; }
    st = dts_oracle_distances(guide, H, W, Cg, sigma_s, sigma_r, dx, dy);        /* O1 */
    if (st) goto done;
    for (int64_t p = 0; p < HW; ++p) {
        const double z = (double)target[p];
        X[p] = z;
        X[HW + p] = z * z;
    }
    st = dts_oracle_dtf(X, H, W, 2, dx, dy, sigma_s, N);                         /* O4 */
    if (st) goto done;
    for (int64_t p = 0; p < HW; ++p) {
        double v = X[HW + p] - X[p] * X[p];                                      /* Eq. 7 */
        if (v < 0.0) v = 0.0;
        if (var) var[p] = v;
        conf[p] = exp(-v / (2.0 * sigma_c * sigma_c));
    }
done:
    free(dx);
    free(dy);
    free(X);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O8: stereo refinement (Eq. 10): gradient descent on
 *     lambda/2 sum (z - zbar)^2 + sum c rho(z - t) + 1/2 sum gamma ||I_L(i) - I_R(i - z_i)||^2
 * with the Charbonnier rho(r) = sqrt(r^2 + eps^2) on the target term.  In the
 * convention of Eq. (3) (reading R23):
 *     g = lambda (z - zbar) + chat rho'(z - t) + gamma sum_k (I_L,k(x) - I_R,k(u)) dI_R,k/dx(u),
 *     rho'(r) = r / sqrt(r^2 + eps^2),   u = x - z   (rectified pair: disparity along the row),
 * I_L = the guide, I_R sampled by linear interpolation along the row; outside
 * [0, W-1] the sample is clamped and its derivative is 0.  chat = c / S as in O6;
 * z^0 = t; z <- z - step g.  guide / right: H x W x Cg fp32 HWC; target, conf: H x W.   */
static void stereo_sample(const float* right, int64_t W, int32_t Cg, int64_t r, double u, int32_t k,
                          double* val, double* slope) {
    const float* row = right + (size_t)r * (size_t)W * (size_t)Cg;
    if (W == 1) { *val = row[k]; *slope = 0.0; return; }
    const int inside = (u >= 0.0 && u <= (double)(W - 1));
    double uc = u < 0.0 ? 0.0 : (u > (double)(W - 1) ? (double)(W - 1) : u);
    int64_t x0 = (int64_t)floor(uc);
    if (x0 > W - 2) x0 = W - 2;
    const double f = uc - (double)x0;
    const double a = row[x0 * Cg + k], b = row[(x0 + 1) * Cg + k];
    *val = (1.0 - f) * a + f * b;
    *slope = inside ? (b - a) : 0.0;
}

int dts_oracle_solve_stereo(const float* guide, const float* right, int64_t H, int64_t W, int32_t Cg,
                            double sigma_s, double sigma_r, int32_t N, const float* target,
                            const float* confidence, double lambda, double step, int32_t iters,
                            double gamma, double eps, int32_t support_mode, double* out) {
    if (!guide || !right || !target || !confidence || !out) return ORACLE_E_ARG;
    if (H < 1 || W < 1 || Cg < 1 || N < 1 || iters < 0 || !(eps > 0.0)) return ORACLE_E_ARG;
    const int64_t HW = H * W;
    double* dx = (double*)malloc(sizeof(double) * (size_t)HW);
    double* dy = (double*)malloc(sizeof(double) * (size_t)HW);
    double* S = (double*)malloc(sizeof(double) * (size_t)HW);
    double* Z = (double*)malloc(sizeof(double) * (size_t)HW);
    double* Zbar = (double*)malloc(sizeof(double) * (size_t)HW);
    double *Ax = NULL, *Ay = NULL;
    int st = ORACLE_OK;
    if (!dx || !dy || !S || !Z || !Zbar) { st = ORACLE_E_OOM; goto done; }
    st = dts_oracle_distances(guide, H, W, Cg, sigma_s, sigma_r, dx, dy);        /* O1 */
    if (st) goto done;
    st = dts_oracle_support(dx, dy, H, W, sigma_s, support_mode, S);            /* O5 */
    if (st) goto done;
    st = make_coefs(dx, dy, H, W, sigma_s, N, &Ax, &Ay);                        /* O2 */
    if (st) goto done;
    for (int64_t p = 0; p < HW; ++p) Z[p] = (double)target[p];
    for (int32_t k = 0; k < iters; ++k) {
        memcpy(Zbar, Z, sizeof(double) * (size_t)HW);
        dtf_with_coefs(Zbar, H, W, 1, N, Ax, Ay);                               /* O4 */
        int64_t p;
#pragma omp parallel for schedule(static)
        for (p = 0; p < HW; ++p) {
            const int64_t r = p / W, x = p % W;
            const double z = Z[p], res = z - (double)target[p];
            const double rho1 = res / sqrt(res * res + eps * eps);              /* Charbonnier */
            double gp = 0.0;
            if (gamma != 0.0) {
                const double u = (double)x - z;
                for (int32_t ch = 0; ch < Cg; ++ch) {
                    double v, sl;
                    stereo_sample(right, W, Cg, r, u, ch, &v, &sl);
                    gp += ((double)guide[(size_t)p * (size_t)Cg + (size_t)ch] - v) * sl;
                }
            }
            const double chat = (double)confidence[p] / S[p];
            Zbar[p] = z - step * (lambda * (z - Zbar[p]) + chat * rho1 + gamma * gp);  /* Eq. (10) step */
        }
        memcpy(Z, Zbar, sizeof(double) * (size_t)HW);
    }
    for (int64_t p = 0; p < HW; ++p) out[p] = Z[p];
done:
    free(dx); free(dy); free(S); free(Z); free(Zbar);
    free(Ax); free(Ay);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O9: depth super-resolution front end (reading R24):
 *   target = bicubic upsampling of the low-resolution depth by an integer factor f
 *            ("simple bicubic interpolation"): Catmull-Rom kernel (a = -0.5),
 *            separable, clamped borders, low-res sample k at high-res coordinate
 *            k f + (f - 1) / 2, i.e. high-res pixel X reads low-res position
 *            u = (X + 0.5) / f - 0.5;
 *   confidence = Gaussian bump around the low-res sample centres (Barron & Poole):
 *            c = exp(-dist^2 / (2 sigma_b^2)), dist = Euclidean distance (high-res pixels)
 *            to the nearest sample centre, sigma_b = f / 4.
 * low: h x w fp32; target, conf: (h f) x (w f) doubles.                               */
static double catmull_rom(double t) {  /* Keys cubic, a = -0.5 */
    t = fabs(t);
    if (t < 1.0) return 1.5 * t * t * t - 2.5 * t * t + 1.0;
    if (t < 2.0) return -0.5 * t * t * t + 2.5 * t * t - 4.0 * t + 2.0;
    return 0.0;
}

int dts_oracle_sr_prepare(const float* low, int64_t h, int64_t w, int32_t f, double* target, double* conf) {
    if (!low || !target || !conf || h < 1 || w < 1 || f < 1) return ORACLE_E_ARG;
    const int64_t H = h * f, W = w * f;
    const double sb = (double)f / 4.0;
    for (int64_t Y = 0; Y < H; ++Y) {
        const double v = ((double)Y + 0.5) / f - 0.5;
        const int64_t j0 = (int64_t)floor(v);
        for (int64_t X = 0; X < W; ++X) {
            const double u = ((double)X + 0.5) / f - 0.5;
            const int64_t i0 = (int64_t)floor(u);
            double acc = 0.0;
            for (int64_t dj = -1; dj <= 2; ++dj) {
                int64_t j = j0 + dj;
                const double wy = catmull_rom(v - (double)j);
                j = j < 0 ? 0 : (j > h - 1 ? h - 1 : j);
                for (int64_t di = -1; di <= 2; ++di) {
                    int64_t i = i0 + di;
                    const double wx = catmull_rom(u - (double)i);
                    i = i < 0 ? 0 : (i > w - 1 ? w - 1 : i);
                    acc += wy * wx * (double)low[j * w + i];
                }
            }
            target[Y * W + X] = acc;
            /* nearest sample centre: k f + (f - 1)/2 with k = clamp(round(u)) */
            int64_t ku = (int64_t)floor(u + 0.5), kv = (int64_t)floor(v + 0.5);
            ku = ku < 0 ? 0 : (ku > w - 1 ? w - 1 : ku);
            kv = kv < 0 ? 0 : (kv > h - 1 ? h - 1 : kv);
            const double ddx = (double)X - ((double)ku * f + (f - 1) / 2.0);
            const double ddy = (double)Y - ((double)kv * f + (f - 1) / 2.0);
            conf[Y * W + X] = exp(-(ddx * ddx + ddy * ddy) / (2.0 * sb * sb));
        }
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* O10: box (normalised-convolution) variant of the edge-aware mean.
 * zbar_i = sum_j W_ij z_j with W_ij = delta{ DT(z_i) - DT(z_j) <= r },
 * read (reading R25, with S:132-160) as the normalised box window on the domain-
 * transform axis:  zbar_i = (1/|N_i|) sum_{j in N_i} z_j,  N_i = { j : |T_j - T_i| <= r },
 * taken along rows (T from the row increments) then columns, N passes with
 * r_i = radius_scale * sigma_i (O2 schedule; radius_scale = sqrt(3), makes the
 * box's standard deviation sigma_i), and the support S_i = |N_i^x| * |N_i^y| at
 * r = radius_scale * sigma_s.
 *
 * Window membership is an integer decision, so both implementations take it in the
 * same precision (reading R25): the increment is evaluated in IEEE single precision in
 * this fixed order (no fused multiply-add, correctly rounded sqrt)
 *     k2 = (sigma_s / sigma_r)^2;  s = sum_k (I_k(c) - I_k(c-1))^2  (k = 0, 1, ...)
 *     d  = sqrt(1 + k2 * s)
 * and the DT coordinate is held in fixed point with 16 fractional bits,
 *     q(c) = round_half_even(d * 2^16)  (capped at 2^30),  T(c) = sum_{c' <= c} q(c'),
 * with the radius R = floor(r * 2^16) computed in double.  Then T is an exact
 * integer and |T_j - T_i| <= R is decided exactly.                          */
#define BOX_QMAX ((int64_t)1 << 30)

static int64_t box_increment(const float* a, const float* b, int32_t C, float k2) {
    float s = 0.0f;
    for (int32_t k = 0; k < C; ++k) {
        float diff = a[k] - b[k];
        float sq = diff * diff;
        s = s + sq;
    }
    float t = k2 * s;
    float v = 1.0f + t;
    float d = sqrtf(v);
    float scaled = d * 65536.0f;
    int64_t q = (int64_t)rintf(scaled);
    return q > BOX_QMAX ? BOX_QMAX : q;
}

/* O10a: fixed-point increments.  qx[r][c] = q between (r, c-1) and (r, c) (qx[r][0] = 0),
 * qy[r][c] = q between (r-1, c) and (r, c) (qy[0][c] = 0).  guide HWC fp32.     */
int dts_oracle_box_increments(const float* guide, int64_t H, int64_t W, int32_t C, float sigma_s,
                              float sigma_r, int64_t* qx, int64_t* qy) {
    if (!guide || !qx || !qy || H < 1 || W < 1 || C < 1) return ORACLE_E_ARG;
    if (!(sigma_s > 0.0f) || !(sigma_r > 0.0f)) return ORACLE_E_ARG;
    const float ratio = sigma_s / sigma_r;
    const float k2 = ratio * ratio;
    for (int64_t r = 0; r < H; ++r)
        for (int64_t c = 0; c < W; ++c) {
            const float* px = guide + (r * W + c) * C;
            qx[r * W + c] = c == 0 ? 0 : box_increment(px, px - C, C, k2);
            qy[r * W + c] = r == 0 ? 0 : box_increment(px, px - W * C, C, k2);
        }
    return ORACLE_OK;
}

/* box radius in fixed point: R = floor(radius_scale * sigma * 2^16), in double */
int64_t dts_oracle_box_radius(double radius_scale, double sigma) {
    return (int64_t)floor(radius_scale * sigma * 65536.0);
}

/* O10b: window of every sample of a line of n samples spaced `stride` apart, from
 * its increments q (q[0] unused): lo = smallest j <= i with T_i - T_j <= R, hi =
 * largest j >= i with T_j - T_i <= R (T is increasing, so N_i = [lo, hi]).
 * lo_off[i] = i - lo, hi_off[i] = hi - i (output spaced like the input).     */
static void box_window_line(const int64_t* q, int64_t n, int64_t stride, int64_t R, int32_t* lo_off,
                            int32_t* hi_off) {
    for (int64_t i = 0; i < n; ++i) {
        int64_t dist = 0, j = i;
        while (j > 0 && dist + q[j * stride] <= R) { dist += q[j * stride]; --j; }   /* T_i - T_{j-1} */
        lo_off[i * stride] = (int32_t)(i - j);
        dist = 0;
        j = i;
        while (j + 1 < n && dist + q[(j + 1) * stride] <= R) { dist += q[(j + 1) * stride]; ++j; }
        hi_off[i * stride] = (int32_t)(j - i);
    }
}

/* windows of all rows (from qx) and all columns (from qy) at radius R            */
int dts_oracle_box_windows(const int64_t* qx, const int64_t* qy, int64_t H, int64_t W, int64_t R,
                           int32_t* lox, int32_t* hix, int32_t* loy, int32_t* hiy) {
    if (!qx || !qy || !lox || !hix || !loy || !hiy || H < 1 || W < 1 || R < 0) return ORACLE_E_ARG;
    int64_t r, c;
#pragma omp parallel for schedule(static)
    for (r = 0; r < H; ++r) box_window_line(qx + r * W, W, 1, R, lox + r * W, hix + r * W);
#pragma omp parallel for schedule(static)
    for (c = 0; c < W; ++c) box_window_line(qy + c, H, W, R, loy + c, hiy + c);
    return ORACLE_OK;
}

/* O10c: the box mean of one line: out_i = (1/(hi-lo+1)) sum_{j=lo}^{hi} x_j, fp64. */
static void box_mean_line(const double* x, double* out, int64_t n, int64_t stride, const int32_t* lo_off,
                          const int32_t* hi_off) {
    for (int64_t i = 0; i < n; ++i) {
        const int64_t lo = i - lo_off[i * stride], hi = i + hi_off[i * stride];
        double sum = 0.0;
        for (int64_t j = lo; j <= hi; ++j) sum += x[j * stride];
        out[i * stride] = sum / (double)(hi - lo + 1);
    }
}

typedef struct {
    int32_t *lox, *hix, *loy, *hiy; /* N x H x W each */
    double* S;                      /* H x W */
} box_tables;

static void box_tables_free(box_tables* b) {
    free(b->lox); free(b->hix); free(b->loy); free(b->hiy); free(b->S);
    memset(b, 0, sizeof(*b));
}

static int box_tables_make(const float* guide, int64_t H, int64_t W, int32_t Cg, float sigma_s, float sigma_r,
                           int32_t N, double radius_scale, int32_t support_mode, box_tables* b) {
    double sig[64];
    memset(b, 0, sizeof(*b));
    if (N < 1 || N > 64) return ORACLE_E_ARG;
    const int64_t HW = H * W;
    int64_t* qx = (int64_t*)malloc(sizeof(int64_t) * (size_t)HW);
    int64_t* qy = (int64_t*)malloc(sizeof(int64_t) * (size_t)HW);
    int32_t* t0 = (int32_t*)malloc(sizeof(int32_t) * (size_t)HW * 4);
    b->lox = (int32_t*)malloc(sizeof(int32_t) * (size_t)HW * (size_t)N);
    b->hix = (int32_t*)malloc(sizeof(int32_t) * (size_t)HW * (size_t)N);
    b->loy = (int32_t*)malloc(sizeof(int32_t) * (size_t)HW * (size_t)N);
    b->hiy = (int32_t*)malloc(sizeof(int32_t) * (size_t)HW * (size_t)N);
    b->S = (double*)malloc(sizeof(double) * (size_t)HW);
    int st = ORACLE_OK;
    if (!qx || !qy || !t0 || !b->lox || !b->hix || !b->loy || !b->hiy || !b->S) { st = ORACLE_E_OOM; goto done; }
    st = dts_oracle_box_increments(guide, H, W, Cg, sigma_s, sigma_r, qx, qy);          /* O10a */
    if (st) goto done;
    dts_oracle_sigmas((double)sigma_s, N, sig);                                         /* O2 */
    for (int32_t i = 0; i < N; ++i) {                                                   /* O10b */
        const int64_t off = (int64_t)i * HW;
        st = dts_oracle_box_windows(qx, qy, H, W, dts_oracle_box_radius(radius_scale, sig[i]), b->lox + off,
                                    b->hix + off, b->loy + off, b->hiy + off);
        if (st) goto done;
    }
    /* support: |N^x| |N^y| at r = radius_scale * sigma_s */
    st = dts_oracle_box_windows(qx, qy, H, W, dts_oracle_box_radius(radius_scale, (double)sigma_s), t0, t0 + HW,
                                t0 + 2 * HW, t0 + 3 * HW);
    if (st) goto done;
    for (int64_t p = 0; p < HW; ++p)
        b->S[p] = support_mode == 1 ? 1.0
                                    : (double)(t0[p] + t0[HW + p] + 1) * (double)(t0[2 * HW + p] + t0[3 * HW + p] + 1);
done:
    free(qx); free(qy); free(t0);
    if (st) box_tables_free(b);
    return st;
}

/* O10d: 2-D box mean: for i = 1..N, rows with the pass-i row windows, then columns
 * with the pass-i column windows (each pass reads the previous pass's output).   */
static void box_dtf_with_tables(double* X, double* tmp, int64_t H, int64_t W, int32_t Ct, int32_t N,
                                const box_tables* b) {
    const int64_t HW = H * W;
    for (int32_t i = 0; i < N; ++i) {
        const int64_t off = (int64_t)i * HW;
        for (int32_t ch = 0; ch < Ct; ++ch) {
            double* P = X + (int64_t)ch * HW;
            int64_t r, c;
#pragma omp parallel for schedule(static)
            for (r = 0; r < H; ++r) box_mean_line(P + r * W, tmp + r * W, W, 1, b->lox + off + r * W, b->hix + off + r * W);
#pragma omp parallel for schedule(static)
            for (c = 0; c < W; ++c) box_mean_line(tmp + c, P + c, H, W, b->loy + off + c, b->hiy + off + c);
        }
    }
}

/* Python-facing: box tables of a guide (windows of every pass, support). */
int dts_oracle_box_tables(const float* guide, int64_t H, int64_t W, int32_t Cg, float sigma_s, float sigma_r,
                          int32_t N, double radius_scale, int32_t* lox, int32_t* hix, int32_t* loy, int32_t* hiy,
                          double* S) {
    if (!guide || !lox || !hix || !loy || !hiy || !S || H < 1 || W < 1 || Cg < 1) return ORACLE_E_ARG;
    box_tables b;
    int st = box_tables_make(guide, H, W, Cg, sigma_s, sigma_r, N, radius_scale, 0, &b);
    if (st) return st;
    const size_t n = sizeof(int32_t) * (size_t)(H * W) * (size_t)N;
    memcpy(lox, b.lox, n); memcpy(hix, b.hix, n); memcpy(loy, b.loy, n); memcpy(hiy, b.hiy, n);
    memcpy(S, b.S, sizeof(double) * (size_t)(H * W));
    box_tables_free(&b);
    return ORACLE_OK;
}

/* Python-facing: the 2-D box mean of Ct planar channels (X in place) for a guide. */
int dts_oracle_box_dtf(double* X, int64_t H, int64_t W, int32_t Ct, const float* guide, int32_t Cg, float sigma_s,
                       float sigma_r, int32_t N, double radius_scale) {
    if (!X || !guide || H < 1 || W < 1 || Ct < 1 || Cg < 1) return ORACLE_E_ARG;
    box_tables b;
    int st = box_tables_make(guide, H, W, Cg, sigma_s, sigma_r, N, radius_scale, 0, &b);
    if (st) return st;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(H * W));
    if (!tmp) { box_tables_free(&b); return ORACLE_E_OOM; }
    box_dtf_with_tables(X, tmp, H, W, Ct, N, &b);
    free(tmp);
    box_tables_free(&b);
    return ORACLE_OK;
}

/* O10e: the DTS iteration of O6 with the box mean (O10d) and the box support. */
int dts_oracle_solve_box(const float* guide, int64_t H, int64_t W, int32_t Cg, float sigma_s, float sigma_r,
                         int32_t N, double radius_scale, const float* target, int32_t Ct, const float* confidence,
                         double lambda, double step, int32_t iters, int32_t support_mode, double* out) {
    if (!guide || !target || !confidence || !out) return ORACLE_E_ARG;
    if (H < 1 || W < 1 || Cg < 1 || Ct < 1 || N < 1 || iters < 0) return ORACLE_E_ARG;
    const int64_t HW = H * W;
    box_tables b;
    int st = box_tables_make(guide, H, W, Cg, sigma_s, sigma_r, N, radius_scale, support_mode, &b);
    if (st) return st;
    double* chat = (double*)malloc(sizeof(double) * (size_t)HW);
    double* Z = (double*)malloc(sizeof(double) * (size_t)HW * (size_t)Ct);
    double* T = (double*)malloc(sizeof(double) * (size_t)HW * (size_t)Ct);
    double* Zbar = (double*)malloc(sizeof(double) * (size_t)HW * (size_t)Ct);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)HW);
    if (!chat || !Z || !T || !Zbar || !tmp) { st = ORACLE_E_OOM; goto done; }
    for (int64_t p = 0; p < HW; ++p) chat[p] = (double)confidence[p] / b.S[p];
    for (int32_t ch = 0; ch < Ct; ++ch)
        for (int64_t p = 0; p < HW; ++p) {
            T[ch * HW + p] = (double)target[p * Ct + ch];
            Z[ch * HW + p] = T[ch * HW + p];
        }
    for (int32_t k = 0; k < iters; ++k) {
        memcpy(Zbar, Z, sizeof(double) * (size_t)HW * (size_t)Ct);
        box_dtf_with_tables(Zbar, tmp, H, W, Ct, N, &b);                            /* O10d */
        int64_t q;
#pragma omp parallel for schedule(static)
        for (q = 0; q < HW * Ct; ++q) {
            int64_t p = q % HW;
            double g = lambda * (Z[q] - Zbar[q]) + chat[p] * (Z[q] - T[q]);        /* Eq. (3) */
            Z[q] = Z[q] - step * g;
        }
    }
    for (int32_t ch = 0; ch < Ct; ++ch)
        for (int64_t p = 0; p < HW; ++p) out[p * Ct + ch] = Z[ch * HW + p];
done:
    free(chat); free(Z); free(T); free(Zbar); free(tmp);
    box_tables_free(&b);
    return st;
}
