/* c_solve.c -- the C ABI used from plain C (no Python, no torch): a seeded synthetic
 * problem on HOST buffers through dts_create / dts_solve_ex / dts_destroy.
 *
 *   gcc -std=c11 -I include examples/c_solve.c -L paper_1805_04590_b200 -ldts_b200 \
 *       -Wl,-rpath,$PWD/paper_1805_04590_b200 -o c_solve
 *   ./c_solve H W C iterations out_prefix
 *
 * Writes <prefix>.guide/.target/.conf (fp32 inputs) and <prefix>.out (fp32 result, H x W)
 * so that a test can run the oracle on the same inputs.  Exit code 0 on success. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "dts.h"

static uint64_t lcg = 0x2545F4914F6CDD1DULL;
static float urand(void) {  /* deterministic uniform [0, 1) */
    lcg = lcg * 6364136223846793005ULL + 1442695040888963407ULL;
    return (float)((lcg >> 40) & 0xFFFFFF) / 16777216.0f;
}

static int dump(const char* prefix, const char* ext, const float* a, size_t n) {
    char name[512];
    snprintf(name, sizeof(name), "%s.%s", prefix, ext);
    FILE* f = fopen(name, "wb");
    if (!f) return 1;
    size_t w = fwrite(a, sizeof(float), n, f);
    fclose(f);
    return w == n ? 0 : 1;
}

int main(int argc, char** argv) {
    if (argc != 6) {
        fprintf(stderr, "usage: %s H W C iterations out_prefix\n", argv[0]);
        return 2;
    }
    const int64_t H = atoll(argv[1]), W = atoll(argv[2]);
    const int32_t C = atoi(argv[3]), iters = atoi(argv[4]);
    const size_t n = (size_t)(H * W);
    float* guide = malloc(sizeof(float) * n * (size_t)C);
    float* target = malloc(sizeof(float) * n);
    float* conf = malloc(sizeof(float) * n);
    float* out = malloc(sizeof(float) * n);
    if (!guide || !target || !conf || !out) return 3;
    for (size_t i = 0; i < n * (size_t)C; ++i) guide[i] = urand();
    for (size_t i = 0; i < n; ++i) {
        target[i] = urand();
        conf[i] = 0.1f + 0.9f * urand();
    }
    dts_ctx* ctx = NULL;
    dts_status st = dts_create(guide, H, W, C, 8.0f, 0.2f, 3, NULL, &ctx);
    if (st != DTS_OK) {
        fprintf(stderr, "dts_create: %s (%s)\n", dts_status_string(st), dts_last_error_string());
        return 4;
    }
    float* resid = malloc(sizeof(float) * (size_t)(iters > 0 ? iters : 1));
    if (!resid) return 3;
    /* step, support_mode, check_inputs, resid_inf_out (per-iteration ||g||_inf, K8) */
    dts_solve_opts opts = {0.99f, 0, 1, resid};
    st = dts_solve_ex(ctx, target, 1, conf, 0.99f, iters, out, NULL, &opts);
    dts_destroy(ctx);
    if (st != DTS_OK) {
        fprintf(stderr, "dts_solve_ex: %s (%s)\n", dts_status_string(st), dts_last_error_string());
        return 5;
    }
    /* an invalid call must come back as a status, not a crash */
    if (dts_create(guide, H, W, C, -1.0f, 0.2f, 3, NULL, &ctx) != DTS_E_ARG) return 6;
    const char* prefix = argv[5];
    if (dump(prefix, "guide", guide, n * (size_t)C) || dump(prefix, "target", target, n) ||
        dump(prefix, "conf", conf, n) || dump(prefix, "out", out, n) || dump(prefix, "resid", resid, (size_t)iters))
        return 7;
    printf("c_solve: %s, %lldx%lld, %d iterations ok\n", dts_version(), (long long)H, (long long)W, iters);
    free(guide);
    free(target);
    free(conf);
    free(out);
    free(resid);
    return 0;
}
