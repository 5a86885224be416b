/*
 * harris_host.c — a plain-C host program using the drop-in C-ABI the way the thesis's
 * generated host code uses its kernel (<name>_init / <name>_run / <name>_destroy over host
 * buffers): no CUDA runtime calls in the application at all.
 *
 * It fills a planar RGB f32 image with the repo's synthetic generator (host restatement
 * in oracle/, linked only as the CHECKER), runs harris_run_host in the exact Appendix-B
 * order and in the default order, and compares against the C oracle:
 *   exact order  -> must be bit-identical
 *   default      -> normalised L-inf within 1e-5
 * Exit status 0 on success.  Build: make -C examples (done by __graft_entry__.build()).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/harris_b200.h"

/* test-infrastructure oracle (oracle/harris_oracle.c) */
void oracle_synth_fill(float* dst, int64_t planes, int64_t rows, int64_t W, int64_t dst_pitch,
                       int64_t dst_plane_stride, int64_t H_global, int64_t row0, int64_t plane0, uint64_t seed,
                       int dist);
int oracle_harris_f32(float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb, int64_t in_pitch,
                      int64_t chan_stride, float kappa, int nthreads);
int oracle_harris_f32_window(float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb,
                             int64_t in_pitch, int64_t chan_stride, float kappa, int nthreads, int window);

int main(int argc, char** argv) {
    const int64_t H = argc > 2 ? atoll(argv[1]) : 1536, W = argc > 2 ? atoll(argv[2]) : 2560;
    const int64_t n = H - 4, m = W - 4;
    float* rgb = malloc(sizeof(float) * 3 * H * W);
    float* out = malloc(sizeof(float) * n * m);
    float* ref = malloc(sizeof(float) * n * m);
    if (!rgb || !out || !ref) return 2;
    oracle_synth_fill(rgb, 3, H, W, W, H * W, H, 0, 0, 12035, 0);
    if (oracle_harris_f32(ref, m, n, m, rgb, W, H * W, 0.04f, 0)) return 3;

    /* options instead of environment variables: evict_normal input loads, plain launches */
    harris_options opts;
    harris_options_default(&opts);
    opts.l2_policy = HARRIS_L2_EVICT_NORMAL;
    opts.pdl = 0;
    harris_ctx* ctx = NULL;
    int rc = harris_init_ex(&ctx, 0, &opts);
    if (rc) {
        fprintf(stderr, "harris_init: %s\n", harris_strerror(rc));
        return 4;
    }
    rc = harris_run_host(ctx, out, m, n, m, rgb, 1, 0.04f, HARRIS_FLAG_EXACT_ORDER);
    if (rc) {
        fprintf(stderr, "harris_run_host: %s (%s)\n", harris_strerror(rc), harris_last_cuda_error(ctx));
        return 5;
    }
    if (memcmp(out, ref, sizeof(float) * n * m) != 0) {
        fprintf(stderr, "exact order differs from the oracle\n");
        return 6;
    }
    rc = harris_run_host(ctx, out, m, n, m, rgb, 1, 0.04f, 0);
    if (rc) return 7;
    double maxd = 0, maxr = 0;
    for (int64_t i = 0; i < n * m; ++i) {
        const double d = fabs((double)out[i] - (double)ref[i]), r = fabs((double)ref[i]);
        if (d > maxd) maxd = d;
        if (r > maxr) maxr = r;
    }
    /* the binomial-window variant (HARRIS_FLAG_BINOMIAL_WINDOW), exact order vs its oracle */
    if (oracle_harris_f32_window(ref, m, n, m, rgb, W, H * W, 0.04f, 0, 1)) return 9;
    rc = harris_run_host(ctx, out, m, n, m, rgb, 1, 0.04f, HARRIS_FLAG_EXACT_ORDER | HARRIS_FLAG_BINOMIAL_WINDOW);
    if (rc) return 10;
    if (memcmp(out, ref, sizeof(float) * n * m) != 0) {
        fprintf(stderr, "binomial window: exact order differs from the oracle\n");
        return 11;
    }
    printf("harris_host %lldx%lld: exact bit-identical, default norm-Linf %.3g, binomial window exact bit-identical, "
           "path %d\n", (long long)H, (long long)W, maxd / (maxr > 0 ? maxr : 1), harris_last_path(ctx));
    harris_destroy(ctx);
    free(rgb);
    free(out);
    free(ref);
    return maxd / (maxr > 0 ? maxr : 1) <= 1e-5 ? 0 : 8;
}
