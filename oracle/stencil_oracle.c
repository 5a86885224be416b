/*
 * stencil_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker for the separable
 * 3x3 stencil of SURVEY.md §8(f) row 3).  Not linked or loaded by the product.
 *
 * The reference package's own stencil workload is the 3x3 binomial filter
 * (binomial.rules:1-27; weights at evalref.py:112-115):
 *   initial  : map (map (dot (join weights2d))) (slide2d 3 1 input)        [direct 2-D]
 *   rewritten: map (\l. map (dot weightsH) (slide 3 1 (map (dot weightsV)
 *                          (transpose l)))) (slide 3 1 input)               [vertical then horizontal]
 * with weights2d = weightsV x weightsH = [1,2,1]^T [1,2,1].  Input (n+2) x (m+2),
 * output n x m, valid region.
 *
 *   oracle_sep3x3_f32 — f32, vertical-then-horizontal order, every product and sum
 *                       rounded (-ffp-contract=off): the GPU EXACT order.
 *   oracle_sep3x3_f64 — f64 in the reference evaluator's order for either form
 *                       (`dot` is CPython >= 3.12's compensated sum, see py_sum in
 *                       harris_oracle.c); pinned bit-for-bit to the evaluator by
 *                       tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline double py_sum3(double a, double b, double c) {
    /* CPython builtin sum over floats with int start 0 (Neumaier), 3 items */
    const double v[3] = {a, b, c};
    double f = 0.0 + v[0], comp = 0.0;
    for (int i = 1; i < 3; ++i) {
        double x = v[i], t = f + x;
        if (fabs(f) >= fabs(x)) comp += (f - t) + x;
        else                    comp += (x - t) + f;
        f = t;
    }
    if (comp != 0.0 && isfinite(comp)) f += comp;
    return f;
}

static inline double py_sum9(const double* v) {
    double f = 0.0 + v[0], comp = 0.0;
    for (int i = 1; i < 9; ++i) {
        double x = v[i], t = f + x;
        if (fabs(f) >= fabs(x)) comp += (f - t) + x;
        else                    comp += (x - t) + f;
        f = t;
    }
    if (comp != 0.0 && isfinite(comp)) f += comp;
    return f;
}

int oracle_sep3x3_f32(float* out, int64_t out_pitch, int64_t n, int64_t m, const float* in,
                      int64_t in_pitch, const float* wv, const float* wh, int nthreads) {
    if (n < 1 || m < 1 || !out || !in || out_pitch < m || in_pitch < m + 2) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < n; ++y) {
        const float* r0 = in + y * in_pitch;
        const float* r1 = r0 + in_pitch;
        const float* r2 = r1 + in_pitch;
        float* o = out + y * out_pitch;
        for (int64_t x = 0; x < m; ++x) {
            float v[3];
            for (int j = 0; j < 3; ++j) {
                float t = 0.0f;
                t = t + wv[0] * r0[x + j];
                t = t + wv[1] * r1[x + j];
                t = t + wv[2] * r2[x + j];
                v[j] = t;
            }
            float s = 0.0f;
            s = s + wh[0] * v[0];
            s = s + wh[1] * v[1];
            s = s + wh[2] * v[2];
            o[x] = s;
        }
    }
    return 0;
}

/* form 0: direct dot(join w2d, join nbh), w2d[i][j] = wv[i]*wh[j];
 * form 1: dot(wh, map (dot wv) (transpose nbh)) (vertical then horizontal) */
int oracle_sep3x3_f64(double* out, int64_t out_pitch, int64_t n, int64_t m, const float* in,
                      int64_t in_pitch, const double* wv, const double* wh, int form, int nthreads) {
    if (n < 1 || m < 1 || !out || !in || out_pitch < m || in_pitch < m + 2) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < n; ++y) {
        const float* r[3] = {in + y * in_pitch, in + (y + 1) * in_pitch, in + (y + 2) * in_pitch};
        double* o = out + y * out_pitch;
        for (int64_t x = 0; x < m; ++x) {
            if (form == 0) {
                double p[9];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) p[3 * i + j] = (wv[i] * wh[j]) * (double)r[i][x + j];
                o[x] = py_sum9(p);
            } else {
                double v[3];
                for (int j = 0; j < 3; ++j)
                    v[j] = py_sum3(wv[0] * (double)r[0][x + j], wv[1] * (double)r[1][x + j],
                                   wv[2] * (double)r[2][x + j]);
                o[x] = py_sum3(wh[0] * v[0], wh[1] * v[1], wh[2] * v[2]);
            }
        }
    }
    return 0;
}
