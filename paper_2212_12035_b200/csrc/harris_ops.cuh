// harris_ops.cuh — the Harris stencil as strip-pipeline ops (strip_pipeline.cuh).
//
// HarrisCore<EXACT> is the per-row register machine shared by every input
// format: given this lane's 4 gray values of input row i (and, for lane 31, the
// 4 gray values of the box's right halo), it updates the rolling 3-row windows
// and produces the 4 coarsity outputs of row i-4.
//   FAST : separable Sobel (horizontal diff / smooth, then vertical), box sums as
//          horizontal shared-pair 3-sums then vertical 3-sums, FMAs, gray already
//          scaled by 1/12 (cbuf+rrot order).
//   EXACT: Appendix-B 9-tap row-major accumulations, never contracted (bit-exact
//          with oracle/harris_oracle.c).
// Slot s2 = R%3 holds row i, s0 = (R+1)%3 row i-2, s1 = (R+2)%3 row i-1.
//
// Input-format ops supply gray:
//   HarrisF32Op : planar RGB f32, 4-D TMA box {132 cols, CH rows, 3 channels, 1 image}
//   HarrisU8Op  : interleaved RGB u8 (HWC, value/255), 3-D TMA box over 32-bit words
//                 {100 words = 400 bytes >= 132 px * 3, CH rows, 1 image}; the byte->float
//                 conversion is fused into the row step.
#pragma once
#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "harris_common.cuh"

namespace harris {

__device__ __forceinline__ void hsum4(const float (&p)[6], float& o0, float& o1, float& o2, float& o3) {
    const float q1 = p[1] + p[2], q3 = p[3] + p[4];
    o0 = p[0] + q1;
    o1 = q1 + p[3];
    o2 = p[2] + q3;
    o3 = q3 + p[5];
}

// products a*b of 6 columns folded into 4 horizontal 3-sums (shared pairs): 8 ops
__device__ __forceinline__ void prodsum4(const float (&a)[6], const float (&b)[6], float& o0, float& o1, float& o2,
                                         float& o3) {
    const float q1 = fmaf(a[1], b[1], a[2] * b[2]);
    const float q3 = fmaf(a[3], b[3], a[4] * b[4]);
    o0 = fmaf(a[0], b[0], q1);
    o1 = fmaf(a[3], b[3], q1);
    o2 = fmaf(a[2], b[2], q3);
    o3 = fmaf(a[5], b[5], q3);
}

// WIN = 1: the binomial window [1,2,1] x [1,2,1] (the reference's weights2d, evalref.py:114-115)
// instead of the 3x3 '+' box — "sometimes used as part of the Harris corner detection instead of
// the 3x3 '+' convolution".  FAST: horizontal [1,2,1] sums of the products,
// vertical fma(2, mid, top + bottom); EXACT: row-major sum from 0 of w * p (oracle wsum9_f32).
// products a*b of 6 columns into 4 horizontal [1,2,1] sums, every product folded into an
// explicit FMA (o = a0 b0 + (2 a1) b1 + a2 b2; 2 a1 is exact): no separate mul + add pair
// exists for ptxas to contract, so both cores produce the same bits
__device__ __forceinline__ void prodwin4(const float (&a)[6], const float (&b)[6], float& o0, float& o1, float& o2,
                                         float& o3) {
    o0 = fmaf(a[0], b[0], fmaf(2.f * a[1], b[1], a[2] * b[2]));
    o1 = fmaf(a[1], b[1], fmaf(2.f * a[2], b[2], a[3] * b[3]));
    o2 = fmaf(a[2], b[2], fmaf(2.f * a[3], b[3], a[4] * b[4]));
    o3 = fmaf(a[3], b[3], fmaf(2.f * a[4], b[4], a[5] * b[5]));
}

template <bool EXACT, int WIN = 0>
struct HarrisCore {
    float kappa;
    // FAST state: horizontal Sobel partials (6 cols) and product 3-sums (3 x 4 cols)
    float D[3][6], Hs[3][6], HB[3][12];
    // EXACT state: gray rows (8 cols) and product rows (3 x 6 cols)
    float G3[3][8], P[3][18];

    __device__ __forceinline__ explicit HarrisCore(float k) : kappa(k) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
            for (int k2 = 0; k2 < 6; ++k2) D[a][k2] = Hs[a][k2] = 0.f;
#pragma unroll
            for (int k2 = 0; k2 < 12; ++k2) HB[a][k2] = 0.f;
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) G3[a][k2] = 0.f;
#pragma unroll
            for (int k2 = 0; k2 < 18; ++k2) P[a][k2] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < 12; ++q) PV[q] = 0.f;
    }

    // lane-halo FAST core with an even stage height: vertical box sums share a row pair —
    // odd row r: PV = H[r-1] + H[r], V = H[r-2] + PV; even row r: V = PV + H[r]
    // (3 adds per 2 rows instead of 4; row parity = R parity because CH is even)
    float PV[12];

    // gown: this lane's 4 gray values; halo(h0..h3) fills the right halo (lane 31 only)
    template <int R, class HaloFn, bool kPairRows = false>
    __device__ __forceinline__ void step(const float (&gown)[4], int lane, HaloFn&& halo, float (&out)[4]) {
        constexpr int s2 = R % 3, s0 = (R + 1) % 3, s1 = (R + 2) % 3;
        constexpr bool kLaneHalo = std::is_same_v<std::decay_t<HaloFn>, NoHalo>;
        static_assert(!(WIN && kLaneHalo && !EXACT), "binomial window: 128-column strips only");
        if constexpr (!EXACT && kLaneHalo) {
            // lane-halo layout: every lane (lane 31 included) has a right neighbour holding
            // the next columns, so Sobel is evaluated on this lane's 4 columns only and the
            // 2 extra columns the box sums need come from lane+1 — the same operands in the
            // same order as computing them here, i.e. bit-identical, 12 FP ops fewer per row
            float gr[6];
#pragma unroll
            for (int k = 0; k < 4; ++k) gr[k] = gown[k];
            gr[4] = __shfl_down_sync(0xffffffffu, gr[0], 1);
            gr[5] = __shfl_down_sync(0xffffffffu, gr[1], 1);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                D[s2][k] = gr[k + 2] - gr[k];
                Hs[s2][k] = fmaf(2.f, gr[k + 1], gr[k]) + gr[k + 2];
            }
            float ix[6], iy[6];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                ix[k] = fmaf(2.f, D[s1][k], D[s0][k] + D[s2][k]);
                iy[k] = Hs[s2][k] - Hs[s0][k];
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                ix[4 + k] = __shfl_down_sync(0xffffffffu, ix[k], 1);
                iy[4 + k] = __shfl_down_sync(0xffffffffu, iy[k], 1);
            }
            prodsum4(ix, ix, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
            prodsum4(ix, iy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
            prodsum4(iy, iy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
            if constexpr (kPairRows) {
                float v[12];
                if constexpr (R % 2 == 1) {
#pragma unroll
                    for (int q = 0; q < 12; ++q) {
                        PV[q] = HB[s1][q] + HB[s2][q];
                        v[q] = HB[s0][q] + PV[q];
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 12; ++q) v[q] = PV[q] + HB[s2][q];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) out[j] = coarsity_fast(v[j], v[4 + j], v[8 + j], kappa);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float sxx = (HB[s0][0 + j] + HB[s1][0 + j]) + HB[s2][0 + j];
                    const float sxy = (HB[s0][4 + j] + HB[s1][4 + j]) + HB[s2][4 + j];
                    const float syy = (HB[s0][8 + j] + HB[s1][8 + j]) + HB[s2][8 + j];
                    out[j] = coarsity_fast(sxx, sxy, syy, kappa);
                }
            }
        } else if constexpr (!EXACT) {
            float gr[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) gr[k] = gown[k];
#pragma unroll
            for (int k = 0; k < 4; ++k) gr[4 + k] = __shfl_down_sync(0xffffffffu, gr[k], 1);
            if constexpr (!std::is_same_v<std::decay_t<HaloFn>, NoHalo>)
                if (lane == 31) halo(gr[4], gr[5], gr[6], gr[7]);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                D[s2][k] = gr[k + 2] - gr[k];
                Hs[s2][k] = fmaf(2.f, gr[k + 1], gr[k]) + gr[k + 2];
            }
            float ix[6], iy[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                ix[k] = fmaf(2.f, D[s1][k], D[s0][k] + D[s2][k]);
                iy[k] = Hs[s2][k] - Hs[s0][k];
            }
            if constexpr (WIN) {
                prodwin4(ix, ix, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
                prodwin4(ix, iy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
                prodwin4(iy, iy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float sxx = fmaf(2.f, HB[s1][0 + j], HB[s0][0 + j] + HB[s2][0 + j]);
                    const float sxy = fmaf(2.f, HB[s1][4 + j], HB[s0][4 + j] + HB[s2][4 + j]);
                    const float syy = fmaf(2.f, HB[s1][8 + j], HB[s0][8 + j] + HB[s2][8 + j]);
                    out[j] = coarsity_fast(sxx, sxy, syy, kappa);
                }
            } else {
                // products folded into the shared-pair horizontal 3-sums with explicit FMAs
                prodsum4(ix, ix, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
                prodsum4(ix, iy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
                prodsum4(iy, iy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float sxx = (HB[s0][0 + j] + HB[s1][0 + j]) + HB[s2][0 + j];
                    const float sxy = (HB[s0][4 + j] + HB[s1][4 + j]) + HB[s2][4 + j];
                    const float syy = (HB[s0][8 + j] + HB[s1][8 + j]) + HB[s2][8 + j];
                    out[j] = coarsity_fast(sxx, sxy, syy, kappa);
                }
            }
        } else {
            const float WX[9] = {-kSobA, 0.f, kSobA, -kSobB, 0.f, kSobB, -kSobA, 0.f, kSobA};
            const float WY[9] = {-kSobA, -kSobB, -kSobA, 0.f, 0.f, 0.f, kSobA, kSobB, kSobA};
            const float W2D[9] = {1.f, 2.f, 1.f, 2.f, 4.f, 2.f, 1.f, 2.f, 1.f};  // binomial window (WIN)
            (void)W2D;
#pragma unroll
            for (int k = 0; k < 4; ++k) G3[s2][k] = gown[k];
#pragma unroll
            for (int k = 0; k < 4; ++k) G3[s2][4 + k] = __shfl_down_sync(0xffffffffu, G3[s2][k], 1);
            if constexpr (!std::is_same_v<std::decay_t<HaloFn>, NoHalo>)
                if (lane == 31) halo(G3[s2][4], G3[s2][5], G3[s2][6], G3[s2][7]);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const float ix = conv9_exact(WX, G3[s0][k], G3[s0][k + 1], G3[s0][k + 2], G3[s1][k], G3[s1][k + 1],
                                             G3[s1][k + 2], G3[s2][k], G3[s2][k + 1], G3[s2][k + 2]);
                const float iy = conv9_exact(WY, G3[s0][k], G3[s0][k + 1], G3[s0][k + 2], G3[s1][k], G3[s1][k + 1],
                                             G3[s1][k + 2], G3[s2][k], G3[s2][k + 1], G3[s2][k + 2]);
                P[s2][k] = __fmul_rn(ix, ix);
                P[s2][6 + k] = __fmul_rn(ix, iy);
                P[s2][12 + k] = __fmul_rn(iy, iy);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float sq[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int o = q * 6 + j;
                    if constexpr (WIN)
                        sq[q] = conv9_exact(W2D, P[s0][o], P[s0][o + 1], P[s0][o + 2], P[s1][o], P[s1][o + 1],
                                            P[s1][o + 2], P[s2][o], P[s2][o + 1], P[s2][o + 2]);
                    else
                        sq[q] = sum9_exact(P[s0][o], P[s0][o + 1], P[s0][o + 2], P[s1][o], P[s1][o + 1],
                                           P[s1][o + 2], P[s2][o], P[s2][o + 1], P[s2][o + 2]);
                }
                out[j] = coarsity_exact(sq[0], sq[1], sq[2], kappa);
            }
        }
    }
};

// gray in the arithmetic of the core: FAST pre-scales by 1/12, EXACT is Appendix B
template <bool EXACT>
__device__ __forceinline__ float gray_of(float r, float g, float b) {
    if constexpr (EXACT)
        return gray_exact(r, g, b);
    else
        return fmaf(kGrayB12, b, fmaf(kGrayG12, g, kGrayR12 * r));
}

// ------------------------------------------------------------ planar RGB f32
template <bool EXACT, int CH, int SC = 128, int WIN = 0>
struct HarrisF32Op {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    using L = Strip<SC>;
    static constexpr int kGroups = 1;
    static constexpr int kStripCols = SC;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kHaloRows = 4;
    static constexpr int kBox = L::kBoxCols;
    static constexpr uint32_t kTxBytes = 3u * CH * kBox * 4u;
    static constexpr uint32_t kStageBytes = (kTxBytes + 127u) / 128u * 128u;
    struct Params {
        float kappa;
    };
    HarrisCore<EXACT, WIN> core;

    __device__ __forceinline__ explicit HarrisF32Op(const Params& p) : core(p.kappa) {}

    __device__ __forceinline__ static void load(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                const int (&col0)[1], int row0, const int (&image)[1],
                                                uint64_t policy) {
        tma_load_4d(smem, tmap, bar, col0[0], row0, 0, image[0], policy);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        const float* sm = reinterpret_cast<const float*>(stage);
        const float* pr = sm + (0 * CH + R) * kBox;
        const float* pg = sm + (1 * CH + R) * kBox;
        const float* pb = sm + (2 * CH + R) * kBox;
        const float4 r = lds128(pr + lane * 4), g = lds128(pg + lane * 4), b = lds128(pb + lane * 4);
        const float gown[4] = {gray_of<EXACT>(r.x, g.x, b.x), gray_of<EXACT>(r.y, g.y, b.y),
                               gray_of<EXACT>(r.z, g.z, b.z), gray_of<EXACT>(r.w, g.w, b.w)};
        if constexpr (L::kLaneHalo) {
            core.template step<R, NoHalo, (CH % 2 == 0)>(gown, lane, NoHalo{}, out[0]);
        } else {
            core.template step<R>(gown, lane, [&](float& h0, float& h1, float& h2, float& h3) {
                const float4 r2 = lds128(pr + kWarpCols), g2 = lds128(pg + kWarpCols), b2 = lds128(pb + kWarpCols);
                h0 = gray_of<EXACT>(r2.x, g2.x, b2.x);
                h1 = gray_of<EXACT>(r2.y, g2.y, b2.y);
                h2 = gray_of<EXACT>(r2.z, g2.z, b2.z);
                h3 = gray_of<EXACT>(r2.w, g2.w, b2.w);
            }, out[0]);
        }
    }
};

// ------------------------------------- planar f32 with row pitch = 2 (mod 4) floats
// Row starts alternate between 16-byte aligned and 8-byte aligned, so TMA cannot address
// single rows — but a PAIR of rows (2P floats) is a 16-byte multiple.  The tensor map views
// each plane as H/2 pair-rows of 2P floats: image row 2j is pair-row j at column x, row
// 2j+1 is pair-row j at column P + x.  A stage of CH = 6 image rows is two boxes of 3
// pair-rows each.  TMA box starts must be 16-byte aligned, so the odd rows' box starts 2
// floats early (P + x0 - 2) and the consumer reads them 2 floats in, with 8-byte loads.
// Scalar lane-halo core (124-column strips), vertical box sums on row pairs.
template <bool EXACT>
struct HarrisF32PairRowOp : HarrisF32Op<EXACT, 6, 124> {
    using Base = HarrisF32Op<EXACT, 6, 124>;
    static constexpr int CH = 6;
    static constexpr bool kSplitStores = true;  // its outputs are typically 2 (mod 4) floats wide
    static constexpr int kRow = 132;                                   // box width (16-byte multiple)
    static constexpr uint32_t kBoxBytes = 3u * 3u * kRow * 4u;         // 3 channels x 3 pair-rows
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;  // TMA destinations: 128-B aligned
    static constexpr uint32_t kTxBytes = 2u * kBoxBytes;
    static constexpr uint32_t kStageBytes = 2u * kBoxStride;
    struct Params {
        float kappa;
        int32_t pitch;  // P: the odd rows' column offset inside a pair-row
    };
    __device__ __forceinline__ explicit HarrisF32PairRowOp(const Params& p) : Base(typename Base::Params{p.kappa}) {}

    __device__ __forceinline__ static void load_p(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                  const int (&col0)[1], int row0, const int (&image)[1],
                                                  uint64_t policy, const Params& p) {
        const int j0 = row0 >> 1;  // row0 is even: tiles start at even rows (planner)
        tma_load_4d(smem, tmap, bar, col0[0], j0, 0, image[0], policy);
        tma_load_4d(static_cast<unsigned char*>(smem) + kBoxStride, tmap, bar, p.pitch + col0[0] - 2, j0, 0,
                    image[0], policy);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        // row R of the stage: parity box R & 1, pair-row R >> 1
        const float* sm = reinterpret_cast<const float*>(stage + (R & 1) * kBoxStride);
        constexpr int rr = R >> 1;
        float c[3][4];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float* q = sm + (ch * 3 + rr) * kRow + 4 * lane;
            if constexpr ((R & 1) == 0) {
                const float4 v = lds128(q);
                c[ch][0] = v.x, c[ch][1] = v.y, c[ch][2] = v.z, c[ch][3] = v.w;
            } else {  // odd rows sit 2 floats into their box
                const float2 v0 = lds64(q + 2), v1 = lds64(q + 4);
                c[ch][0] = v0.x, c[ch][1] = v0.y, c[ch][2] = v1.x, c[ch][3] = v1.y;
            }
        }
        const float gown[4] = {gray_of<EXACT>(c[0][0], c[1][0], c[2][0]), gray_of<EXACT>(c[0][1], c[1][1], c[2][1]),
                               gray_of<EXACT>(c[0][2], c[1][2], c[2][2]), gray_of<EXACT>(c[0][3], c[1][3], c[2][3])};
        // no row-pair box sums: FAST stays bit-identical to the other f32 paths
        this->core.template step<R, NoHalo, false>(gown, lane, NoHalo{}, out[0]);
    }
};

// ------------------------------------------------- planar f32 with an odd row pitch
// The pair-row idea one level up: 4 rows (4P floats) are a 16-byte multiple.  The tensor
// map views each plane as H/4 quad-rows; image row 4j + r is quad-row j at column rP + x.
// A stage of CH = 12 rows is four boxes (one per r) of 3 quad-rows.  Each class's box starts
// s_r = rP mod 4 floats early (16-byte aligned) and the consumer reads it s_r floats in
// (s_0 = 0: 16-byte loads; otherwise scalar loads at a warp-uniform skew).
template <bool EXACT>
struct HarrisF32QuadRowOp : HarrisF32Op<EXACT, 12, 124> {
    using Base = HarrisF32Op<EXACT, 12, 124>;
    static constexpr int CH = 12;
    static constexpr int kRow = 132;
    static constexpr uint32_t kBoxBytes = 3u * 3u * kRow * 4u;
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kTxBytes = 4u * kBoxBytes;
    static constexpr uint32_t kStageBytes = 4u * kBoxStride;
    struct Params {
        float kappa;
        int32_t pitch;  // P (odd)
    };
    int skew[4];  // s_r: float offset of class r's data in its box

    __device__ __forceinline__ explicit HarrisF32QuadRowOp(const Params& p) : Base(typename Base::Params{p.kappa}) {
#pragma unroll
        for (int r = 0; r < 4; ++r) skew[r] = (r * p.pitch) & 3;
    }

    __device__ __forceinline__ static void load_p(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                  const int (&col0)[1], int row0, const int (&image)[1],
                                                  uint64_t policy, const Params& p) {
        const int j0 = row0 >> 2;  // row0 is a multiple of 4 (planner)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int x = r * p.pitch;
            tma_load_4d(static_cast<unsigned char*>(smem) + r * kBoxStride, tmap, bar, x - (x & 3) + col0[0], j0, 0,
                        image[0], policy);
        }
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        constexpr int cls = R & 3, qr = R >> 2;
        const float* sm = reinterpret_cast<const float*>(stage + cls * kBoxStride);
        float c[3][4];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float* q = sm + (ch * 3 + qr) * kRow + 4 * lane;
            if constexpr (cls == 0) {
                const float4 v = lds128(q);
                c[ch][0] = v.x, c[ch][1] = v.y, c[ch][2] = v.z, c[ch][3] = v.w;
            } else if constexpr (cls == 2) {  // 2P = 2 (mod 4): 8-byte aligned
                const float2 v0 = lds64(q + 2), v1 = lds64(q + 4);
                c[ch][0] = v0.x, c[ch][1] = v0.y, c[ch][2] = v1.x, c[ch][3] = v1.y;
            } else {  // skew 1 or 3 (warp-uniform): scalar + 8-byte + scalar
                const int s = skew[cls];
                const float2 v = lds64(q + s + 1);
                c[ch][0] = q[s], c[ch][1] = v.x, c[ch][2] = v.y, c[ch][3] = q[s + 3];
            }
        }
        const float gown[4] = {gray_of<EXACT>(c[0][0], c[1][0], c[2][0]), gray_of<EXACT>(c[0][1], c[1][1], c[2][1]),
                               gray_of<EXACT>(c[0][2], c[1][2], c[2][2]), gray_of<EXACT>(c[0][3], c[1][3], c[2][3])};
        // no row-pair box sums: FAST stays bit-identical to the other f32 paths
        this->core.template step<R, NoHalo, false>(gown, lane, NoHalo{}, out[0]);
    }
};

// --------------------------------------------------- interleaved RGB u8 (HWC)
// byte k of w as an exact float: 0x4B0000bb is 2^23 + b, minus 2^23 (PRMT + FADD)
__device__ __forceinline__ float u8f(uint32_t w, int k) {
    return __int_as_float(__byte_perm(w, 0x4B000000u, 0x7440u | uint32_t(k))) - 8388608.0f;
}

// FAST gray of raw bytes: weights pre-scaled by 1/(12*255); EXACT: Appendix-B gray of
// the IEEE quotients v/255 (the same f32 values the planar path sees for u8/255 data)
template <bool EXACT>
__device__ __forceinline__ float gray_u8(float r, float g, float b) {
    if constexpr (EXACT) {
        return gray_exact(__fdiv_rn(r, 255.0f), __fdiv_rn(g, 255.0f), __fdiv_rn(b, 255.0f));
    } else {
        constexpr float kR = 0.299f / (12.0f * 255.0f), kG = 0.587f / (12.0f * 255.0f),
                        kB = 0.114f / (12.0f * 255.0f);
        return fmaf(kB, b, fmaf(kG, g, kR * r));
    }
}

// 4 pixels = 12 bytes = 3 words: w0 = R0 G0 B0 R1, w1 = G1 B1 R2 G2, w2 = B2 R3 G3 B3
// FAST: N = 299 R + 587 G + 114 B exactly in integers — two IDP.2A (16-bit weights x
// byte pairs) per pixel straight on the interleaved words, no byte extraction — summed
// onto 0x4B000000 so the bit pattern is the float 2^23 + N (N <= 255000 < 2^23); then
// gray = fma(2^23 + N, s, -s * 2^23) = RN(s * N), s = 1/(12 * 255 * 1000) (the Sobel 1/12
// folded in).  One rounding, so it is closer to the f64 oracle than the three-FMA form.
constexpr float kGrayU8Scale = 1.0f / (12.0f * 255.0f * 1000.0f);
__device__ __forceinline__ void gray4_u8_bits(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t& n0, uint32_t& n1,
                                              uint32_t& n2, uint32_t& n3) {
    constexpr uint32_t kRG = 299u | (587u << 16), kB0 = 114u, k0R = 299u << 16, kGB = 587u | (114u << 16);
    constexpr uint32_t kBias = 0x4B000000u;
    n0 = __dp2a_hi(kB0, w0, __dp2a_lo(kRG, w0, kBias));   // R0 G0 | B0
    n1 = __dp2a_lo(kGB, w1, __dp2a_hi(k0R, w0, kBias));   // R1 | G1 B1
    n2 = __dp2a_lo(kB0, w2, __dp2a_hi(kRG, w1, kBias));   // R2 G2 | B2
    n3 = __dp2a_hi(kGB, w2, __dp2a_lo(k0R, w2, kBias));   // R3 | G3 B3
}
__device__ __forceinline__ float gray_u8_from_bits(uint32_t n) {
    return fmaf(__uint_as_float(n), kGrayU8Scale, -kGrayU8Scale * 8388608.0f);
}

template <bool EXACT>
__device__ __forceinline__ void gray4_u8(uint32_t w0, uint32_t w1, uint32_t w2, float& g0, float& g1, float& g2,
                                         float& g3) {
    if constexpr (EXACT) {
        g0 = gray_u8<EXACT>(u8f(w0, 0), u8f(w0, 1), u8f(w0, 2));
        g1 = gray_u8<EXACT>(u8f(w0, 3), u8f(w1, 0), u8f(w1, 1));
        g2 = gray_u8<EXACT>(u8f(w1, 2), u8f(w1, 3), u8f(w2, 0));
        g3 = gray_u8<EXACT>(u8f(w2, 1), u8f(w2, 2), u8f(w2, 3));
    } else {
        uint32_t n0, n1, n2, n3;
        gray4_u8_bits(w0, w1, w2, n0, n1, n2, n3);
        g0 = gray_u8_from_bits(n0);
        g1 = gray_u8_from_bits(n1);
        g2 = gray_u8_from_bits(n2);
        g3 = gray_u8_from_bits(n3);
    }
}

template <bool EXACT, int CH, int SC = 128>
struct HarrisU8Op {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    using L = Strip<SC>;
    static constexpr int kGroups = 1;
    static constexpr int kStripCols = SC;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kHaloRows = 4;
    static constexpr int kWords = L::kU8BoxWords;
    static constexpr uint32_t kTxBytes = uint32_t(CH) * kWords * 4u;
    static constexpr uint32_t kStageBytes = (kTxBytes + 127u) / 128u * 128u;
    struct Params {
        float kappa;
    };
    HarrisCore<EXACT> core;

    __device__ __forceinline__ explicit HarrisU8Op(const Params& p) : core(p.kappa) {}

    // tensor map over 32-bit words: {ceil(3W/4) words, H rows, B images}
    __device__ __forceinline__ static void load(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                const int (&col0)[1], int row0, const int (&image)[1],
                                                uint64_t policy) {
        tma_load_3d(smem, tmap, bar, L::u8_box_word(col0[0] / SC), row0, image[0], policy);
    }

    int skip = 0;  // words before the strip's first pixel in the box (SC = 124 only)
    __device__ __forceinline__ void begin_tile(const int (&col0)[1], int, const int (&)[1]) {
        if constexpr (SC != 128) skip = L::u8_skip(col0[0] / SC);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(stage) + R * kWords + skip;
        float gown[4];
        gray4_u8<EXACT>(w[3 * lane], w[3 * lane + 1], w[3 * lane + 2], gown[0], gown[1], gown[2], gown[3]);
        if constexpr (L::kLaneHalo) {
            core.template step<R, NoHalo, (CH % 2 == 0)>(gown, lane, NoHalo{}, out[0]);
        } else {
            core.template step<R>(gown, lane, [&](float& h0, float& h1, float& h2, float& h3) {
                gray4_u8<EXACT>(w[96], w[97], w[98], h0, h1, h2, h3);
            }, out[0]);
        }
    }
};

}  // namespace harris
