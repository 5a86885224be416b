/*
 * harris_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * Nothing in the product path (paper_2212_12035_b200/, include/) links, loads or
 * calls this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker or as the
 * timed CPU arm.
 *
 * It is a plain-C restatement of the Harris corner detector the thesis optimises
 * (arXiv 2212.12035, /root/reference/PAPER.md), in two precisions:
 *
 *   oracle_harris_f32  — the f32 arithmetic contract of SURVEY.md Appendix B,
 *                        i.e. the op order of the Shine-generated cbuf OpenCL
 *                        kernel (PAPER.md:4587-4590 gray, 4613-4635 Sobel 9-tap
 *                        accumulation from 0 in row-major order incl. zero
 *                        taps, 4697-4728 box sums of products accumulated from 0,
 *                        4730 coarsity).  Compile with -ffp-contract=off so no
 *                        a*b+c is fused: every product and sum is rounded to f32.
 *   oracle_harris_f64  — the same algorithm in f64 with the exact evaluation
 *                        order of the reference package's evaluator on the Rise
 *                        program (sges evalref.py:110-111 `dot` = Python sum from
 *                        0; evalref.py:53-63 `reduce add 0` = left fold;
 *                        SURVEY.md Appendix A term).  It is pinned bit-for-bit
 *                        against /root/reference's own evaluator by
 *                        tests/golden/ (fixtures made by
 *                        tests/golden/make_golden.py).
 *
 * Structure follows the thesis cbuf schedule:
 * the output is split into 32-row strips processed in parallel (OpenMP), each
 * strip keeps 3-line circular buffers of gray, of Ix/Iy and of the three
 * products, so every stage is computed once per pixel and inner loops run along
 * a row (vectorisable; no reassociation because no -ffast-math).
 *
 * Layout (Rise type harris : 3.(n+4).(m+4).f32 -> n.m.f32):
 *   rgb  element (c, y, x) at rgb[c*chan_stride + y*in_pitch + x], H=n+4, W=m+4
 *   out  element (y, x)    at out[y*out_pitch + x]
 *
 * Synthetic inputs: oracle_synth_fill reproduces the product's device generator
 * (paper_2212_12035_b200/csrc/harris_synth.cu) so the checker can regenerate any
 * shard of any bench image on the host.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define STRIP 32

/* ---------------------------------------------------------------- synth --- */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* dst element (p, y, x) at dst[p*dst_plane_stride + y*dst_pitch + x] holds the
 * value of global plane (plane0+p), global row (row0+y) of an image stack with
 * H_global rows and W columns.  dist 0: U[0,1) with 24-bit mantissa;
 * dist 1: u8/255.  Keyed by the global linear index so any band regenerates
 * identically. */
void oracle_synth_fill(float* dst, int64_t planes, int64_t rows, int64_t W,
                       int64_t dst_pitch, int64_t dst_plane_stride,
                       int64_t H_global, int64_t row0, int64_t plane0,
                       uint64_t seed, int dist) {
    const uint64_t key = seed * 0xD1B54A32D192ED03ULL;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t p = 0; p < planes; ++p) {
        for (int64_t y = 0; y < rows; ++y) {
            float* row = dst + p * dst_plane_stride + y * dst_pitch;
            uint64_t base = ((uint64_t)(plane0 + p) * (uint64_t)H_global
                             + (uint64_t)(row0 + y)) * (uint64_t)W;
            for (int64_t x = 0; x < W; ++x) {
                uint64_t z = mix64(base + (uint64_t)x + key);
                row[x] = dist == 1 ? (float)(z >> 56) / 255.0f
                                   : (float)(z >> 40) * 0x1p-24f;
            }
        }
    }
}

/* ------------------------------------------------------------ f32 oracle --- */
static const float GR = 0.299f, GG = 0.587f, GB = 0.114f;
static const float SA = 0.083333336f, SB = 0.16666667f;

static void gray_line_f32(float* g, const float* r, const float* gg, const float* b,
                          int64_t W) {
    for (int64_t x = 0; x < W; ++x) {
        float t = 0.0f;                      /* t4 = 0; t4 += 0.299*R; ... */
        t = t + GR * r[x];
        t = t + GG * gg[x];
        t = t + GB * b[x];
        g[x] = t;
    }
}

/* Ix and Iy for one row from gray rows g0,g1,g2. */
static void sobel_line_f32(float* ix, float* iy, const float* g0, const float* g1,
                           const float* g2, int64_t Ws) {
    for (int64_t x = 0; x < Ws; ++x) {
        float t = 0.0f;
        t = t + (-SA) * g0[x];  t = t + 0.0f * g0[x + 1];  t = t + SA * g0[x + 2];
        t = t + (-SB) * g1[x];  t = t + 0.0f * g1[x + 1];  t = t + SB * g1[x + 2];
        t = t + (-SA) * g2[x];  t = t + 0.0f * g2[x + 1];  t = t + SA * g2[x + 2];
        ix[x] = t;
        float u = 0.0f;
        u = u + (-SA) * g0[x];  u = u + (-SB) * g0[x + 1]; u = u + (-SA) * g0[x + 2];
        u = u + 0.0f * g1[x];   u = u + 0.0f * g1[x + 1];  u = u + 0.0f * g1[x + 2];
        u = u + SA * g2[x];     u = u + SB * g2[x + 1];    u = u + SA * g2[x + 2];
        iy[x] = u;
    }
}

static void products_line_f32(float* pxx, float* pxy, float* pyy, const float* ix,
                              const float* iy, int64_t Ws) {
    for (int64_t x = 0; x < Ws; ++x) {
        pxx[x] = ix[x] * ix[x];
        pxy[x] = ix[x] * iy[x];
        pyy[x] = iy[x] * iy[x];
    }
}

/* the reference's binomial window weights2d = [[1,2,1],[2,4,2],[1,2,1]] (evalref.py:114-115),
 * the "binomial filter instead of the 3x3 '+' convolution" Harris variant:
 * S = dot(join weights2d, join window) = row-major sum from 0 of w*p (w*p exact in f32) */
static inline float wsum9_f32(const float* a, const float* b, const float* c, int64_t x) {
    float s = 0.0f;
    s = s + 1.0f * a[x]; s = s + 2.0f * a[x + 1]; s = s + 1.0f * a[x + 2];
    s = s + 2.0f * b[x]; s = s + 4.0f * b[x + 1]; s = s + 2.0f * b[x + 2];
    s = s + 1.0f * c[x]; s = s + 2.0f * c[x + 1]; s = s + 1.0f * c[x + 2];
    return s;
}

static inline float sum9_f32(const float* a, const float* b, const float* c, int64_t x) {
    float s = 0.0f;
    s = s + a[x]; s = s + a[x + 1]; s = s + a[x + 2];
    s = s + b[x]; s = s + b[x + 1]; s = s + b[x + 2];
    s = s + c[x]; s = s + c[x + 1]; s = s + c[x + 2];
    return s;
}

int oracle_harris_f32_window(float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb,
                             int64_t in_pitch, int64_t chan_stride, float kappa, int nthreads, int window);

/* one 32-row strip of the cbuf schedule; buf: 3W + 15Ws floats of per-thread line buffers */
static void cbuf_strip_f32_w(float* buf, float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb,
                             int64_t in_pitch, int64_t chan_stride, float kappa, int64_t s, int window) {
    const int64_t W = m + 4, Ws = m + 2;
    float* gl[3] = {buf, buf + W, buf + 2 * W};
    float* sb = buf + 3 * W;
    float *ix[3], *iy[3], *pxx[3], *pxy[3], *pyy[3];
    for (int k = 0; k < 3; ++k) {
        ix[k] = sb + (0 + k) * Ws;  iy[k] = sb + (3 + k) * Ws;
        pxx[k] = sb + (6 + k) * Ws; pxy[k] = sb + (9 + k) * Ws;
        pyy[k] = sb + (12 + k) * Ws;
    }
    const int64_t y0 = s * STRIP;
    const int64_t y1 = (y0 + STRIP < n) ? y0 + STRIP : n;
    /* input rows y0 .. y1+3; gray row r lives in gl[r % 3]; Sobel row
     * q (= gray rows q..q+2) lives in slot q % 3 */
    for (int64_t r = y0; r < y1 + 4; ++r) {
        const float* R = rgb + 0 * chan_stride + r * in_pitch;
        const float* G = rgb + 1 * chan_stride + r * in_pitch;
        const float* B = rgb + 2 * chan_stride + r * in_pitch;
        gray_line_f32(gl[r % 3], R, G, B, W);
        if (r >= y0 + 2) {
            int64_t q = r - 2;
            int k = (int)(q % 3);
            sobel_line_f32(ix[k], iy[k], gl[q % 3], gl[(q + 1) % 3],
                           gl[(q + 2) % 3], Ws);
            products_line_f32(pxx[k], pxy[k], pyy[k], ix[k], iy[k], Ws);
        }
        if (r >= y0 + 4) {
            int64_t y = r - 4;
            int a = (int)(y % 3), b = (int)((y + 1) % 3), c = (int)((y + 2) % 3);
            float* o = out + y * out_pitch;
            for (int64_t x = 0; x < m; ++x) {
                float sxx = window ? wsum9_f32(pxx[a], pxx[b], pxx[c], x) : sum9_f32(pxx[a], pxx[b], pxx[c], x);
                float sxy = window ? wsum9_f32(pxy[a], pxy[b], pxy[c], x) : sum9_f32(pxy[a], pxy[b], pxy[c], x);
                float syy = window ? wsum9_f32(pyy[a], pyy[b], pyy[c], x) : sum9_f32(pyy[a], pyy[b], pyy[c], x);
                float det = sxx * syy - sxy * sxy;
                float tr = sxx + syy;
                o[x] = det - kappa * tr * tr;
            }
        }
    }
}

static void cbuf_strip_f32(float* buf, float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb,
                           int64_t in_pitch, int64_t chan_stride, float kappa, int64_t s) {
    cbuf_strip_f32_w(buf, out, out_pitch, n, m, rgb, in_pitch, chan_stride, kappa, s, 0);
}

#define CBUF_BUF_FLOATS(W, Ws) ((size_t)(3 * (W) + 15 * (Ws)))

int oracle_harris_f32(float* out, int64_t out_pitch, int64_t n, int64_t m,
                      const float* rgb, int64_t in_pitch, int64_t chan_stride,
                      float kappa, int nthreads) {
    return oracle_harris_f32_window(out, out_pitch, n, m, rgb, in_pitch, chan_stride, kappa, nthreads, 0);
}

/* window 0: the 3x3 '+' box sums (Appendix B); 1: the reference's binomial window */
int oracle_harris_f32_window(float* out, int64_t out_pitch, int64_t n, int64_t m,
                             const float* rgb, int64_t in_pitch, int64_t chan_stride,
                             float kappa, int nthreads, int window) {
    if (n < 1 || m < 1 || !out || !rgb || out_pitch < m || in_pitch < m + 4) return -1;
    const int64_t W = m + 4, Ws = m + 2;
    const int64_t nstrips = (n + STRIP - 1) / STRIP;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        /* per-thread circular line buffers: 3 gray, 3 Ix, 3 Iy, 3x3 products */
        float* buf = (float*)malloc(sizeof(float) * CBUF_BUF_FLOATS(W, Ws));
        if (!buf) {
#pragma omp atomic write
            err = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < nstrips; ++s)
            if (buf) cbuf_strip_f32_w(buf, out, out_pitch, n, m, rgb, in_pitch, chan_stride, kappa, s, window);
        free(buf);
    }
    return err;
}

/* ------------------------------------------------------------ f64 oracle --- */
/* Same schedule, f64 arithmetic, evaluation order of sges eval_term on the
 * Appendix-A Rise term: `dot` is Python's builtin sum over the products
 * (evalref.py:110-111), `reduce add 0` is a plain left fold (evalref.py:53-63),
 * det = a*c + (-1)*(b*b), out = det + (-1)*((k*tr)*tr).
 *
 * CPython >= 3.12 sums floats with Neumaier compensation (builtin_sum_impl in
 * Python/bltinmodule.c): the int start 0 is added to the first item exactly,
 * the remaining items are accumulated with a running compensation c, and c is
 * added once at the end when it is non-zero and finite.  py_sum reproduces that
 * bit-for-bit, which is what makes this f64 oracle identical to the reference
 * evaluator (tests/golden/). */
static inline double py_sum(const double* v, int k) {
    double f = 0.0 + v[0];   /* int 0 + first float item */
    double c = 0.0;
    for (int i = 1; i < k; ++i) {
        double x = v[i];
        double t = f + x;
        if (fabs(f) >= fabs(x)) c += (f - t) + x;
        else                    c += (x - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

static const double DGR = 0.299, DGG = 0.587, DGB = 0.114;
#define DA (1.0 / 12.0)
#define DB (2.0 / 12.0)

int oracle_harris_f64_window(double* out, int64_t out_pitch, int64_t n, int64_t m,
                             const float* rgb, int64_t in_pitch, int64_t chan_stride,
                             double kappa, int nthreads, int window);

int oracle_harris_f64(double* out, int64_t out_pitch, int64_t n, int64_t m,
                      const float* rgb, int64_t in_pitch, int64_t chan_stride,
                      double kappa, int nthreads) {
    return oracle_harris_f64_window(out, out_pitch, n, m, rgb, in_pitch, chan_stride, kappa, nthreads, 0);
}

/* window 0: `+3x3` = map (map (reduce add 0)) over the 3x3 neighbourhood (a left fold from 0);
 * window 1: the binomial window = dot (join weights2d) (evalref.py:110-111, 114-115): Python
 * sum of w*p in row-major order, i.e. py_sum (Neumaier-compensated, Python >= 3.12) */
int oracle_harris_f64_window(double* out, int64_t out_pitch, int64_t n, int64_t m,
                             const float* rgb, int64_t in_pitch, int64_t chan_stride,
                             double kappa, int nthreads, int window) {
    if (n < 1 || m < 1 || !out || !rgb || out_pitch < m || in_pitch < m + 4) return -1;
    const int64_t W = m + 4, Ws = m + 2;
    const int64_t nstrips = (n + STRIP - 1) / STRIP;
    const double wsx[9] = {-DA, 0.0, DA, -DB, 0.0, DB, -DA, 0.0, DA};
    const double wsy[9] = {-DA, -DB, -DA, 0.0, 0.0, 0.0, DA, DB, DA};
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        double* buf = (double*)malloc(sizeof(double) * (size_t)(3 * W + 15 * Ws));
        if (!buf) {
#pragma omp atomic write
            err = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < nstrips; ++s) {
            if (!buf) continue;
            double* gl[3] = {buf, buf + W, buf + 2 * W};
            double* sb = buf + 3 * W;
            double *ix[3], *iy[3], *pxx[3], *pxy[3], *pyy[3];
            for (int k = 0; k < 3; ++k) {
                ix[k] = sb + (0 + k) * Ws;  iy[k] = sb + (3 + k) * Ws;
                pxx[k] = sb + (6 + k) * Ws; pxy[k] = sb + (9 + k) * Ws;
                pyy[k] = sb + (12 + k) * Ws;
            }
            const int64_t y0 = s * STRIP;
            const int64_t y1 = (y0 + STRIP < n) ? y0 + STRIP : n;
            for (int64_t r = y0; r < y1 + 4; ++r) {
                const float* R = rgb + 0 * chan_stride + r * in_pitch;
                const float* G = rgb + 1 * chan_stride + r * in_pitch;
                const float* B = rgb + 2 * chan_stride + r * in_pitch;
                double* g = gl[r % 3];
                for (int64_t x = 0; x < W; ++x) {
                    const double v[3] = {DGR * (double)R[x], DGG * (double)G[x],
                                         DGB * (double)B[x]};
                    g[x] = py_sum(v, 3);
                }
                if (r >= y0 + 2) {
                    int64_t q = r - 2;
                    int k = (int)(q % 3);
                    const double* rows[3] = {gl[q % 3], gl[(q + 1) % 3], gl[(q + 2) % 3]};
                    for (int64_t x = 0; x < Ws; ++x) {
                        double vx[9], vy[9];
                        for (int i = 0; i < 3; ++i)
                            for (int j = 0; j < 3; ++j) {
                                vx[3 * i + j] = wsx[3 * i + j] * rows[i][x + j];
                                vy[3 * i + j] = wsy[3 * i + j] * rows[i][x + j];
                            }
                        double t = py_sum(vx, 9), u = py_sum(vy, 9);
                        ix[k][x] = t;
                        iy[k][x] = u;
                        pxx[k][x] = t * t;
                        pxy[k][x] = t * u;
                        pyy[k][x] = u * u;
                    }
                }
                if (r >= y0 + 4) {
                    int64_t y = r - 4;
                    int a = (int)(y % 3), b = (int)((y + 1) % 3), c = (int)((y + 2) % 3);
                    double* o = out + y * out_pitch;
                    static const double w2d[9] = {1.0, 2.0, 1.0, 2.0, 4.0, 2.0, 1.0, 2.0, 1.0};
                    for (int64_t x = 0; x < m; ++x) {
                        double sxx = 0.0, sxy = 0.0, syy = 0.0;
                        const int rr[3] = {a, b, c};
                        if (window) {
                            double vxx[9], vxy[9], vyy[9];
                            for (int i = 0; i < 3; ++i)
                                for (int j = 0; j < 3; ++j) {
                                    vxx[3 * i + j] = w2d[3 * i + j] * pxx[rr[i]][x + j];
                                    vxy[3 * i + j] = w2d[3 * i + j] * pxy[rr[i]][x + j];
                                    vyy[3 * i + j] = w2d[3 * i + j] * pyy[rr[i]][x + j];
                                }
                            sxx = py_sum(vxx, 9);
                            sxy = py_sum(vxy, 9);
                            syy = py_sum(vyy, 9);
                        } else {
                            for (int i = 0; i < 3; ++i)
                                for (int j = 0; j < 3; ++j) {
                                    sxx = sxx + pxx[rr[i]][x + j];
                                    sxy = sxy + pxy[rr[i]][x + j];
                                    syy = syy + pyy[rr[i]][x + j];
                                }
                        }
                        double det = sxx * syy + (-1.0) * (sxy * sxy);
                        double tr = sxx + syy;
                        o[x] = det + (-1.0) * ((kappa * tr) * tr);
                    }
                }
            }
        }
        free(buf);
    }
    return err;
}

/* ----------------------------------------------- f32 cbuf+rrot CPU port --- */
/* The thesis's fastest CPU schedule, cbuf+rrot (1.24x over
 * cbuf on ARM): 32-row strips, 3-line circular buffers of gray,
 * SEPARATED convolutions — vertical [1,2,1] / [-1,0,1] sums of gray, then the
 * horizontal +-1/12, 1/6 taps — and box sums as vertical
 * 3-row sums of the products followed by horizontal 3-sums,
 * every accumulation from 0 in listing order (-ffp-contract=off).  A different
 * op order from Appendix B (results agree within the SURVEY.md §8(d) tolerance,
 * not bit-for-bit); used as the strongest CPU baseline. */
/* vertical 3-row sums of the products; a separate function with
 * restrict line pointers so gcc vectorises it like the cbuf line functions */
static void rrot_vbox_line_f32(float* restrict vxx, float* restrict vxy, float* restrict vyy,
                               const float* restrict a0, const float* restrict a1, const float* restrict a2,
                               const float* restrict b0, const float* restrict b1, const float* restrict b2,
                               int64_t Ws) {
    for (int64_t x = 0; x < Ws; ++x) {
        float t = 0.0f;
        t = t + a0[x] * a0[x]; t = t + a1[x] * a1[x]; t = t + a2[x] * a2[x];
        vxx[x] = t;
        float u = 0.0f;
        u = u + a0[x] * b0[x]; u = u + a1[x] * b1[x]; u = u + a2[x] * b2[x];
        vxy[x] = u;
        float v = 0.0f;
        v = v + b0[x] * b0[x]; v = v + b1[x] * b1[x]; v = v + b2[x] * b2[x];
        vyy[x] = v;
    }
}

/* one 32-row strip of the cbuf+rrot schedule; buf: 5W + 9Ws floats */
static void rrot_strip_f32(float* buf, float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb,
                           int64_t in_pitch, int64_t chan_stride, float kappa, int64_t s) {
    const int64_t W = m + 4, Ws = m + 2;
    float* gl[3] = {buf, buf + W, buf + 2 * W};
    float* vs = buf + 3 * W;          /* vertical [1,2,1] sum, width W */
    float* vd = buf + 4 * W;          /* vertical [-1,0,1] diff, width W */
    float* sb = buf + 5 * W;
    float *ix[3], *iy[3];
    for (int k = 0; k < 3; ++k) { ix[k] = sb + k * Ws; iy[k] = sb + (3 + k) * Ws; }
    float* vxx = sb + 6 * Ws;
    float* vxy = sb + 7 * Ws;
    float* vyy = sb + 8 * Ws;
    const int64_t y0 = s * STRIP;
    const int64_t y1 = (y0 + STRIP < n) ? y0 + STRIP : n;
    for (int64_t r = y0; r < y1 + 4; ++r) {
        const float* R = rgb + 0 * chan_stride + r * in_pitch;
        const float* G = rgb + 1 * chan_stride + r * in_pitch;
        const float* B = rgb + 2 * chan_stride + r * in_pitch;
        gray_line_f32(gl[r % 3], R, G, B, W);
        if (r >= y0 + 2) {
            const int64_t q = r - 2;
            const float* g0 = gl[q % 3];
            const float* g1 = gl[(q + 1) % 3];
            const float* g2 = gl[(q + 2) % 3];
            for (int64_t x = 0; x < W; ++x) {
                float t = 0.0f;
                t += 1.0f * g0[x]; t += 2.0f * g1[x]; t += 1.0f * g2[x];
                vs[x] = t;
                float u = 0.0f;
                u += -1.0f * g0[x]; u += 0.0f * g1[x]; u += 1.0f * g2[x];
                vd[x] = u;
            }
            float* px = ix[q % 3];
            float* py = iy[q % 3];
            for (int64_t x = 0; x < Ws; ++x) {
                float t = 0.0f;
                t = t + (-SA) * vs[x]; t = t + 0.0f * vs[x + 1]; t = t + SA * vs[x + 2];
                px[x] = t;
                float u = 0.0f;
                u = u + SA * vd[x]; u = u + SB * vd[x + 1]; u = u + SA * vd[x + 2];
                py[x] = u;
            }
        }
        if (r >= y0 + 4) {
            const int64_t y = r - 4;
            rrot_vbox_line_f32(vxx, vxy, vyy, ix[y % 3], ix[(y + 1) % 3], ix[(y + 2) % 3],
                               iy[y % 3], iy[(y + 1) % 3], iy[(y + 2) % 3], Ws);
            float* o = out + y * out_pitch;
            for (int64_t x = 0; x < m; ++x) {
                float sxy = 0.0f; sxy = sxy + vxy[x]; sxy = sxy + vxy[x + 1]; sxy = sxy + vxy[x + 2];
                float syy = 0.0f; syy = syy + vyy[x]; syy = syy + vyy[x + 1]; syy = syy + vyy[x + 2];
                float sxx = 0.0f; sxx = sxx + vxx[x]; sxx = sxx + vxx[x + 1]; sxx = sxx + vxx[x + 2];
                o[x] = sxx * syy - sxy * sxy - kappa * (sxx + syy) * (sxx + syy);
            }
        }
    }
}

#define RROT_BUF_FLOATS(W, Ws) ((size_t)(5 * (W) + 9 * (Ws)))

int oracle_harris_f32_rrot(float* out, int64_t out_pitch, int64_t n, int64_t m,
                           const float* rgb, int64_t in_pitch, int64_t chan_stride,
                           float kappa, int nthreads) {
    if (n < 1 || m < 1 || !out || !rgb || out_pitch < m || in_pitch < m + 4) return -1;
    const int64_t W = m + 4, Ws = m + 2;
    const int64_t nstrips = (n + STRIP - 1) / STRIP;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        /* 3 gray lines, 2 vertical-sum lines, 3 Ix + 3 Iy lines, 3 vertical box lines */
        float* buf = (float*)malloc(sizeof(float) * RROT_BUF_FLOATS(W, Ws));
        if (!buf) {
#pragma omp atomic write
            err = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < nstrips; ++s)
            if (buf) rrot_strip_f32(buf, out, out_pitch, n, m, rgb, in_pitch, chan_stride, kappa, s);
        free(buf);
    }
    return err;
}

/* batched forms: contiguous 3 x H x W images, contiguous n x m outputs.  One OpenMP
 * loop over every (image, strip) pair, so a batch of small images keeps every core busy
 * (per-image loops leave cores idle when strips per image is not a multiple of threads). */
typedef void (*strip_fn)(float*, float*, int64_t, int64_t, int64_t, const float*, int64_t, int64_t, float, int64_t);

static int batched_strips(strip_fn fn, size_t buf_floats, float* out, int64_t n, int64_t m, const float* rgb,
                          int64_t batch, float kappa, int nthreads) {
    if (n < 1 || m < 1 || batch < 1 || !out || !rgb) return -1;
    const int64_t H = n + 4, W = m + 4;
    const int64_t nstrips = (n + STRIP - 1) / STRIP;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        float* buf = (float*)malloc(sizeof(float) * buf_floats);
        if (!buf) {
#pragma omp atomic write
            err = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < batch * nstrips; ++t) {
            const int64_t b = t / nstrips, s = t - b * nstrips;
            if (buf) fn(buf, out + b * n * m, m, n, m, rgb + b * 3 * H * W, W, H * W, kappa, s);
        }
        free(buf);
    }
    return err;
}

int oracle_harris_f32_rrot_batched(float* out, int64_t n, int64_t m, const float* rgb,
                                   int64_t batch, float kappa, int nthreads) {
    return batched_strips(rrot_strip_f32, RROT_BUF_FLOATS(m + 4, m + 2), out, n, m, rgb, batch, kappa, nthreads);
}

int oracle_harris_f32_batched(float* out, int64_t n, int64_t m, const float* rgb,
                              int64_t batch, float kappa, int nthreads) {
    return batched_strips(cbuf_strip_f32, CBUF_BUF_FLOATS(m + 4, m + 2), out, n, m, rgb, batch, kappa, nthreads);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
