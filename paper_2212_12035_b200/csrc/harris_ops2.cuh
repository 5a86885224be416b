// harris_ops2.cuh — dual-strip Harris ops with packed FP32x2 arithmetic.
//
// A tile is TWO adjacent 128-column strips (kGroups = 2): lane l owns columns
// [4l, 4l+4) of strip A and the same columns of strip B.  Every operation of the
// Harris row step is identical for A and B, so the pair (A, B) is carried in one
// float2 and evaluated with sm_100's packed instructions (__ffma2_rn /
// __fadd2_rn / __fmul2_rn -> FFMA2 / FADD2 / FMUL2): half the FP instructions per
// pixel of the scalar core, which keeps the kernel HBM-bound even when the SM
// clock drops under the power cap (the scalar core becomes per-warp-latency
// bound there; tools/variance.py).
//
// Arithmetic is the same contract as harris_ops.cuh:
//   FAST : separable Sobel, fused product+pair-sum box rows, FMAs.
//   EXACT: Appendix-B 9-tap orders, component-wise scalar __fmul_rn/__fadd_rn
//          (see xadd2 below for why not the packed forms), bit-exact with the oracle.
// In FAST, a - b is evaluated as fma(b, -1, a): one rounding of the exact
// difference, i.e. identical to FSUB.
#pragma once
#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "harris_common.cuh"
#include "harris_ops.cuh"

namespace harris {

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, f2(-1.0f), a); }

__device__ __forceinline__ float2 shfl_down2(float2 v) {
    return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

// exact Appendix-B pieces on pairs.  ptxas (CUDA 12.9, sm_100a) packs paired
// mul.rn/add.rn into FMUL2/FADD2 and then contracts them into FFMA2 despite the
// explicit rounding modifier (observed in SASS), which breaks bit-exactness.  The
// multiplies are therefore written as fma(a, b, -0), which is bit-identical to a
// rounded product and cannot be fused with the following add.  EXACT is the parity
// path, so its speed is irrelevant.
__device__ __forceinline__ float2 xadd2(float2 a, float2 b) {
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
// a*b as fma(a, b, -0): bit-identical to round(a*b) (adding -0 preserves every value
// and sign), and an fma can never be contracted with the following add
__device__ __forceinline__ float2 xmul2(float2 a, float2 b) {
    return make_float2(__fmaf_rn(a.x, b.x, -0.0f), __fmaf_rn(a.y, b.y, -0.0f));
}
__device__ __forceinline__ float2 xsub2(float2 a, float2 b) {
    return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
}

__device__ __forceinline__ float2 gray_exact2(float2 r, float2 g, float2 b) {
    float2 t = xadd2(f2(0.0f), xmul2(f2(kGrayR), r));
    t = xadd2(t, xmul2(f2(kGrayG), g));
    return xadd2(t, xmul2(f2(kGrayB), b));
}

__device__ __forceinline__ float2 conv9_exact2(const float (&w)[9], float2 a0, float2 a1, float2 a2, float2 b0,
                                               float2 b1, float2 b2, float2 c0, float2 c1, float2 c2) {
    float2 t = f2(0.0f);
    t = xadd2(t, xmul2(f2(w[0]), a0));
    t = xadd2(t, xmul2(f2(w[1]), a1));
    t = xadd2(t, xmul2(f2(w[2]), a2));
    t = xadd2(t, xmul2(f2(w[3]), b0));
    t = xadd2(t, xmul2(f2(w[4]), b1));
    t = xadd2(t, xmul2(f2(w[5]), b2));
    t = xadd2(t, xmul2(f2(w[6]), c0));
    t = xadd2(t, xmul2(f2(w[7]), c1));
    t = xadd2(t, xmul2(f2(w[8]), c2));
    return t;
}

__device__ __forceinline__ float2 sum9_exact2(float2 a0, float2 a1, float2 a2, float2 b0, float2 b1, float2 b2,
                                              float2 c0, float2 c1, float2 c2) {
    float2 s = xadd2(f2(0.0f), a0);
    s = xadd2(s, a1);
    s = xadd2(s, a2);
    s = xadd2(s, b0);
    s = xadd2(s, b1);
    s = xadd2(s, b2);
    s = xadd2(s, c0);
    s = xadd2(s, c1);
    return xadd2(s, c2);
}

__device__ __forceinline__ float2 coarsity_exact2(float2 sxx, float2 sxy, float2 syy, float k) {
    const float2 det = xsub2(xmul2(sxx, syy), xmul2(sxy, sxy));
    const float2 tr = xadd2(sxx, syy);
    return xsub2(det, xmul2(xmul2(f2(k), tr), tr));
}

template <bool EXACT, int WIN = 0>  // WIN: the binomial window (harris_ops.cuh)
struct HarrisCore2 {
    float kappa;
    float2 D[3][6], Hs[3][6], HB[3][12];   // FAST
    float2 G3[3][8], P[3][18];             // EXACT

    __device__ __forceinline__ explicit HarrisCore2(float k) : kappa(k) {
#pragma unroll
        for (int q = 0; q < 12; ++q) PV[q] = f2(0.f);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
            for (int j = 0; j < 6; ++j) D[a][j] = Hs[a][j] = f2(0.f);
#pragma unroll
            for (int j = 0; j < 12; ++j) HB[a][j] = f2(0.f);
#pragma unroll
            for (int j = 0; j < 8; ++j) G3[a][j] = f2(0.f);
#pragma unroll
            for (int j = 0; j < 18; ++j) P[a][j] = f2(0.f);
        }
    }

    // products a*b of 6 columns folded into 4 horizontal 3-sums (shared pairs)
    __device__ __forceinline__ static void prodsum4(const float2 (&a)[6], const float2 (&b)[6], float2& o0,
                                                    float2& o1, float2& o2, float2& o3) {
        const float2 q1 = fma2(a[1], b[1], mul2(a[2], b[2]));
        const float2 q3 = fma2(a[3], b[3], mul2(a[4], b[4]));
        o0 = fma2(a[0], b[0], q1);
        o1 = fma2(a[3], b[3], q1);
        o2 = fma2(a[2], b[2], q3);
        o3 = fma2(a[5], b[5], q3);
    }

    // products a*b of 6 columns into 4 horizontal [1,2,1] sums (binomial window), the same
    // explicit-FMA form as the scalar core's prodwin4
    __device__ __forceinline__ static void prodwin4(const float2 (&a)[6], const float2 (&b)[6], float2& o0,
                                                    float2& o1, float2& o2, float2& o3) {
        o0 = fma2(a[0], b[0], fma2(mul2(f2(2.f), a[1]), b[1], mul2(a[2], b[2])));
        o1 = fma2(a[1], b[1], fma2(mul2(f2(2.f), a[2]), b[2], mul2(a[3], b[3])));
        o2 = fma2(a[2], b[2], fma2(mul2(f2(2.f), a[3]), b[3], mul2(a[4], b[4])));
        o3 = fma2(a[3], b[3], fma2(mul2(f2(2.f), a[4]), b[4], mul2(a[5], b[5])));
    }

    // gown: (A, B) gray of this lane's 4 columns; halo(h0..h3) fills the right halo of
    // both strips for lane 31
    float2 PV[12];  // row-pair partial box sums (kPairRows: the u8 op, where rounding parity
                    // with the f32 paths is not required and instructions are the bound)

    template <int R, class HaloFn, bool kPairRows = false>
    __device__ __forceinline__ void step(const float2 (&gown)[4], int lane, HaloFn&& halo, float (&out)[2][4]) {
        constexpr int s2 = R % 3, s0 = (R + 1) % 3, s1 = (R + 2) % 3;
        constexpr bool kLaneHalo = std::is_same_v<std::decay_t<HaloFn>, NoHalo>;
        // lane-halo layout, FAST: Sobel on this lane's 4 columns only, columns 4 and 5 from
        // lane + 1 (same operands, same order: bit-identical; 24 fewer state registers)
        constexpr int NC = (kLaneHalo && !EXACT) ? 4 : 6;
        float2 g[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = gown[k];
#pragma unroll
        for (int k = 0; k < NC - 2; ++k) g[4 + k] = shfl_down2(g[k]);
        if constexpr (!kLaneHalo)
            if (lane == 31) halo(g[4], g[5], g[6], g[7]);
        if constexpr (!EXACT) {
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                D[s2][k] = sub2(g[k + 2], g[k]);
                Hs[s2][k] = add2(fma2(f2(2.f), g[k + 1], g[k]), g[k + 2]);
            }
            float2 ix[6], iy[6];
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                ix[k] = fma2(f2(2.f), D[s1][k], add2(D[s0][k], D[s2][k]));
                iy[k] = sub2(Hs[s2][k], Hs[s0][k]);
            }
            if constexpr (NC == 4) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    ix[4 + k] = shfl_down2(ix[k]);
                    iy[4 + k] = shfl_down2(iy[k]);
                }
            }
            static_assert(!WIN || (NC == 6 && !kPairRows), "binomial window: 128-column strips, 3-row sums");
            if constexpr (WIN) {
                prodwin4(ix, ix, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
                prodwin4(ix, iy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
                prodwin4(iy, iy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
            } else {
                prodsum4(ix, ix, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
                prodsum4(ix, iy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
                prodsum4(iy, iy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
            }
            const float2 nk = f2(-kappa);
            float2 v[12];
            if constexpr (WIN) {
#pragma unroll
                for (int q = 0; q < 12; ++q) v[q] = fma2(f2(2.f), HB[s1][q], add2(HB[s0][q], HB[s2][q]));
            } else if constexpr (kPairRows) {
                // odd row r: PV = H[r-1] + H[r], V = H[r-2] + PV; even row: V = PV + H[r]
                if constexpr (R % 2 == 1) {
#pragma unroll
                    for (int q = 0; q < 12; ++q) {
                        PV[q] = add2(HB[s1][q], HB[s2][q]);
                        v[q] = add2(HB[s0][q], PV[q]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 12; ++q) v[q] = add2(PV[q], HB[s2][q]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 12; ++q) v[q] = add2(add2(HB[s0][q], HB[s1][q]), HB[s2][q]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 sxx = v[0 + j], sxy = v[4 + j], syy = v[8 + j];
                // same op order as the scalar core's coarsity_fast, so FAST results are
                // bit-identical across every kernel path / configuration
                const float2 det = fma2(make_float2(-sxy.x, -sxy.y), sxy, mul2(sxx, syy));
                const float2 tr = add2(sxx, syy);
                const float2 o = fma2(mul2(nk, tr), tr, det);
                out[0][j] = o.x;
                out[1][j] = o.y;
            }
        } else {
            const float WX[9] = {-kSobA, 0.f, kSobA, -kSobB, 0.f, kSobB, -kSobA, 0.f, kSobA};
            const float WY[9] = {-kSobA, -kSobB, -kSobA, 0.f, 0.f, 0.f, kSobA, kSobB, kSobA};
            const float W2D[9] = {1.f, 2.f, 1.f, 2.f, 4.f, 2.f, 1.f, 2.f, 1.f};  // binomial window (WIN)
            (void)W2D;
#pragma unroll
            for (int k = 0; k < 8; ++k) G3[s2][k] = g[k];
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const float2 ix = conv9_exact2(WX, G3[s0][k], G3[s0][k + 1], G3[s0][k + 2], G3[s1][k],
                                               G3[s1][k + 1], G3[s1][k + 2], G3[s2][k], G3[s2][k + 1], G3[s2][k + 2]);
                const float2 iy = conv9_exact2(WY, G3[s0][k], G3[s0][k + 1], G3[s0][k + 2], G3[s1][k],
                                               G3[s1][k + 1], G3[s1][k + 2], G3[s2][k], G3[s2][k + 1], G3[s2][k + 2]);
                P[s2][k] = xmul2(ix, ix);
                P[s2][6 + k] = xmul2(ix, iy);
                P[s2][12 + k] = xmul2(iy, iy);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 sq[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int o = q * 6 + j;
                    if constexpr (WIN)
                        sq[q] = conv9_exact2(W2D, P[s0][o], P[s0][o + 1], P[s0][o + 2], P[s1][o], P[s1][o + 1],
                                             P[s1][o + 2], P[s2][o], P[s2][o + 1], P[s2][o + 2]);
                    else
                        sq[q] = sum9_exact2(P[s0][o], P[s0][o + 1], P[s0][o + 2], P[s1][o], P[s1][o + 1],
                                            P[s1][o + 2], P[s2][o], P[s2][o + 1], P[s2][o + 2]);
                }
                const float2 o = coarsity_exact2(sq[0], sq[1], sq[2], kappa);
                out[0][j] = o.x;
                out[1][j] = o.y;
            }
        }
    }
};

template <bool EXACT>
__device__ __forceinline__ float2 gray2_of(float2 r, float2 g, float2 b) {
    if constexpr (EXACT)
        return gray_exact2(r, g, b);
    else
        return fma2(f2(kGrayB12), b, fma2(f2(kGrayG12), g, mul2(f2(kGrayR12), r)));
}

// ------------------------------------------------------------ planar RGB f32
// Two TMA boxes per stage ({132 cols, CH rows, 3 channels, 1 image} at x and x+128).
template <bool EXACT, int CH, int SC = 128, int WIN = 0>
struct HarrisF32x2Op {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    using L = Strip<SC>;
    static constexpr bool kCacheProducer = false;  // measured: per-stage decode is faster here
    static constexpr int kGroups = 2;
    static constexpr int kStripCols = SC;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kHaloRows = 4;
    static constexpr int kBox = L::kBoxCols;
    static constexpr uint32_t kBoxBytes = 3u * CH * kBox * 4u;
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kTxBytes = 2u * kBoxBytes;
    static constexpr uint32_t kStageBytes = 2u * kBoxStride;
    struct Params {
        float kappa;
    };
    HarrisCore2<EXACT, WIN> core;

    __device__ __forceinline__ explicit HarrisF32x2Op(const Params& p) : core(p.kappa) {}

    // one box per strip (the two strips may belong to different images)
    __device__ __forceinline__ static void load(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                const int (&col0)[2], int row0, const int (&image)[2],
                                                uint64_t policy) {
        tma_load_4d(smem, tmap, bar, col0[0], row0, 0, image[0], policy);
        tma_load_4d(static_cast<unsigned char*>(smem) + kBoxStride, tmap, bar, col0[1], row0, 0, image[1], policy);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[2][4]) {
        const float* a = reinterpret_cast<const float*>(stage);
        const float* b = reinterpret_cast<const float*>(stage + kBoxStride);
        const int o_r = (0 * CH + R) * kBox, o_g = (1 * CH + R) * kBox, o_b = (2 * CH + R) * kBox;
        const float4 ra = lds128(a + o_r + lane * 4), ga = lds128(a + o_g + lane * 4), ba = lds128(a + o_b + lane * 4);
        const float4 rb = lds128(b + o_r + lane * 4), gb = lds128(b + o_g + lane * 4), bb = lds128(b + o_b + lane * 4);
        // gray in scalar form: the results can be allocated straight into the (A, B)
        // register pairs, where packed gray would first need MOVs to pair the inputs
        const float2 gown[4] = {
            make_float2(gray_of<EXACT>(ra.x, ga.x, ba.x), gray_of<EXACT>(rb.x, gb.x, bb.x)),
            make_float2(gray_of<EXACT>(ra.y, ga.y, ba.y), gray_of<EXACT>(rb.y, gb.y, bb.y)),
            make_float2(gray_of<EXACT>(ra.z, ga.z, ba.z), gray_of<EXACT>(rb.z, gb.z, bb.z)),
            make_float2(gray_of<EXACT>(ra.w, ga.w, ba.w), gray_of<EXACT>(rb.w, gb.w, bb.w))};
        if constexpr (L::kLaneHalo) {
            core.template step<R>(gown, lane, NoHalo{}, out);
        } else if (adjacent) {
            float hA[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) hA[k] = __shfl_sync(0xffffffffu, gown[k].y, 0);
            core.template step<R>(gown, lane, [&](float2& h0, float2& h1, float2& h2, float2& h3) {
                const float4 r2b = lds128(b + o_r + kWarpCols), g2b = lds128(b + o_g + kWarpCols),
                             b2b = lds128(b + o_b + kWarpCols);
                h0 = make_float2(hA[0], gray_of<EXACT>(r2b.x, g2b.x, b2b.x));
                h1 = make_float2(hA[1], gray_of<EXACT>(r2b.y, g2b.y, b2b.y));
                h2 = make_float2(hA[2], gray_of<EXACT>(r2b.z, g2b.z, b2b.z));
                h3 = make_float2(hA[3], gray_of<EXACT>(r2b.w, g2b.w, b2b.w));
            }, out);
        } else {
            core.template step<R>(gown, lane, [&](float2& h0, float2& h1, float2& h2, float2& h3) {
                const float4 r2a = lds128(a + o_r + kWarpCols), g2a = lds128(a + o_g + kWarpCols),
                             b2a = lds128(a + o_b + kWarpCols);
                const float4 r2b = lds128(b + o_r + kWarpCols), g2b = lds128(b + o_g + kWarpCols),
                             b2b = lds128(b + o_b + kWarpCols);
                h0 = make_float2(gray_of<EXACT>(r2a.x, g2a.x, b2a.x), gray_of<EXACT>(r2b.x, g2b.x, b2b.x));
                h1 = make_float2(gray_of<EXACT>(r2a.y, g2a.y, b2a.y), gray_of<EXACT>(r2b.y, g2b.y, b2b.y));
                h2 = make_float2(gray_of<EXACT>(r2a.z, g2a.z, b2a.z), gray_of<EXACT>(r2b.z, g2b.z, b2b.z));
                h3 = make_float2(gray_of<EXACT>(r2a.w, g2a.w, b2a.w), gray_of<EXACT>(r2b.w, g2b.w, b2b.w));
            }, out);
        }
    }

    bool adjacent = false;  // strip B is strip A + 1 of the same image (per tile)
    __device__ __forceinline__ void begin_tile(const int (&col0)[2], int, const int (&image)[2]) {
        adjacent = image[0] == image[1] && col0[1] == col0[0] + SC;
    }
};

// --------------------------------------------------- interleaved RGB u8 (HWC)
// (byte k of wa, byte k of wb) as exact floats: PRMT each, one FADD2 for both
__device__ __forceinline__ float2 u8f2(uint32_t wa, uint32_t wb, int k) {
    const float2 m = make_float2(__int_as_float(__byte_perm(wa, 0x4B000000u, 0x7440u | uint32_t(k))),
                                 __int_as_float(__byte_perm(wb, 0x4B000000u, 0x7440u | uint32_t(k))));
    return add2(m, f2(-8388608.0f));
}

template <bool EXACT>
__device__ __forceinline__ float2 gray2_u8(float2 r, float2 g, float2 b) {
    if constexpr (EXACT) {
        const float2 q255 = f2(255.0f);
        return gray_exact2(make_float2(__fdiv_rn(r.x, q255.x), __fdiv_rn(r.y, q255.y)),
                           make_float2(__fdiv_rn(g.x, q255.x), __fdiv_rn(g.y, q255.y)),
                           make_float2(__fdiv_rn(b.x, q255.x), __fdiv_rn(b.y, q255.y)));
    } else {
        constexpr float kR = 0.299f / (12.0f * 255.0f), kG = 0.587f / (12.0f * 255.0f),
                        kB = 0.114f / (12.0f * 255.0f);
        return fma2(f2(kB), b, fma2(f2(kG), g, mul2(f2(kR), r)));
    }
}

// 4 pixels of strips A and B from their 3 words each
template <bool EXACT>
__device__ __forceinline__ void gray4_u8x2(const uint32_t (&a)[3], const uint32_t (&b)[3], float2& g0, float2& g1,
                                           float2& g2, float2& g3) {
    if constexpr (!EXACT) {
        // strips A and B: integer gray sums (harris_ops.cuh gray4_u8_bits), one FFMA2 per pair
        uint32_t na[4], nb[4];
        gray4_u8_bits(a[0], a[1], a[2], na[0], na[1], na[2], na[3]);
        gray4_u8_bits(b[0], b[1], b[2], nb[0], nb[1], nb[2], nb[3]);
        const float2 s = f2(kGrayU8Scale), c = f2(-kGrayU8Scale * 8388608.0f);
        g0 = fma2(make_float2(__uint_as_float(na[0]), __uint_as_float(nb[0])), s, c);
        g1 = fma2(make_float2(__uint_as_float(na[1]), __uint_as_float(nb[1])), s, c);
        g2 = fma2(make_float2(__uint_as_float(na[2]), __uint_as_float(nb[2])), s, c);
        g3 = fma2(make_float2(__uint_as_float(na[3]), __uint_as_float(nb[3])), s, c);
        return;
    }
    g0 = gray2_u8<EXACT>(u8f2(a[0], b[0], 0), u8f2(a[0], b[0], 1), u8f2(a[0], b[0], 2));
    g1 = gray2_u8<EXACT>(u8f2(a[0], b[0], 3), u8f2(a[1], b[1], 0), u8f2(a[1], b[1], 1));
    g2 = gray2_u8<EXACT>(u8f2(a[1], b[1], 2), u8f2(a[1], b[1], 3), u8f2(a[2], b[2], 0));
    g3 = gray2_u8<EXACT>(u8f2(a[2], b[2], 1), u8f2(a[2], b[2], 2), u8f2(a[2], b[2], 3));
}

template <bool EXACT, int CH, int SC = 128>
struct HarrisU8x2Op {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    static constexpr bool kTwoStoreVariants = true;  // issue-bound: measured +5.6 %
    using L = Strip<SC>;
    static constexpr int kGroups = 2;
    static constexpr int kStripCols = SC;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kHaloRows = 4;
    static constexpr int kWords = L::kU8BoxWords;
    static constexpr uint32_t kBoxBytes = uint32_t(CH) * kWords * 4u;
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kTxBytes = 2u * kBoxBytes;
    static constexpr uint32_t kStageBytes = 2u * kBoxStride;
    struct Params {
        float kappa;
    };
    HarrisCore2<EXACT> core;

    __device__ __forceinline__ explicit HarrisU8x2Op(const Params& p) : core(p.kappa) {}

    // tensor map over 32-bit words; strip cs starts at word 96 * cs
    __device__ __forceinline__ static void load(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                const int (&col0)[2], int row0, const int (&image)[2],
                                                uint64_t policy) {
        tma_load_3d(smem, tmap, bar, L::u8_box_word(col0[0] / SC), row0, image[0], policy);
        tma_load_3d(static_cast<unsigned char*>(smem) + kBoxStride, tmap, bar, L::u8_box_word(col0[1] / SC), row0,
                    image[1], policy);
    }

    int skip_a = 0, skip_b = 0;  // words before each strip's first pixel (SC = 124 only)
    __device__ __forceinline__ void begin_tile(const int (&col0)[2], int, const int (&)[2]) {
        if constexpr (SC != 128) {
            skip_a = L::u8_skip(col0[0] / SC);
            skip_b = L::u8_skip(col0[1] / SC);
        }
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[2][4]) {
        const uint32_t* wa = reinterpret_cast<const uint32_t*>(stage) + R * kWords + skip_a;
        const uint32_t* wb = reinterpret_cast<const uint32_t*>(stage + kBoxStride) + R * kWords + skip_b;
        const uint32_t a[3] = {wa[3 * lane], wa[3 * lane + 1], wa[3 * lane + 2]};
        const uint32_t b[3] = {wb[3 * lane], wb[3 * lane + 1], wb[3 * lane + 2]};
        float2 gown[4];
        gray4_u8x2<EXACT>(a, b, gown[0], gown[1], gown[2], gown[3]);
        if constexpr (L::kLaneHalo) {
            core.template step<R, NoHalo, (CH % 2 == 0)>(gown, lane, NoHalo{}, out);
        } else {
            core.template step<R>(gown, lane, [&](float2& h0, float2& h1, float2& h2, float2& h3) {
                const uint32_t ha[3] = {wa[96], wa[97], wa[98]};
                const uint32_t hb[3] = {wb[96], wb[97], wb[98]};
                gray4_u8x2<EXACT>(ha, hb, h0, h1, h2, h3);
            }, out);
        }
    }
};

// ------------------------------ interleaved u8 whose row pitch is 4, 8 or 12 (mod 16) bytes
// (e.g. 1080 or 1366 px wide: 3W % 16 != 0, so TMA cannot step single rows).  K rows (K = 2
// for pitch = 8 mod 16, 4 for pitch = 4 mod 8) are a 16-byte multiple: the tensor map views
// each image as H/K group-rows of K*P bytes (32-bit words), image row K*j + r is group-row j
// at word r*P/4 + x.  A stage of CH rows is, per strip, K boxes (one per row class r) of
// CH/K group-rows, each starting at its 16-byte aligned-down word and read `skip` words in
// (a per-tile constant per class and strip).  Packed dual-strip u8 core as the TMA path.
template <bool EXACT, int K>
struct HarrisU8RowGroupOp {
    static_assert(K == 2 || K == 4, "row groups of 2 or 4");
    static constexpr bool kTwoStoreVariants = true;  // measured +1.2 % (the f32 TMA op: -1.5 %)
    static constexpr int CH = K == 2 ? 6 : 12;
    using L = Strip<124>;
    static constexpr int kGroups = 2;
    static constexpr int kStripCols = 124;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kHaloRows = 4;
    static constexpr int kWords = L::kU8BoxWords;
    static constexpr int kBoxRows = CH / K;  // group-rows per box
    static constexpr uint32_t kBoxBytes = uint32_t(kBoxRows) * kWords * 4u;
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kTxBytes = 2u * K * kBoxBytes;
    static constexpr uint32_t kStageBytes = 2u * K * kBoxStride;
    struct Params {
        float kappa;
        int32_t pitch_words;  // P / 4
    };
    HarrisCore2<EXACT> core;
    int32_t pw;
    int skip_a[K], skip_b[K];

    __device__ __forceinline__ explicit HarrisU8RowGroupOp(const Params& p) : core(p.kappa), pw(p.pitch_words) {}

    __device__ __forceinline__ static void load_p(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                  const int (&col0)[2], int row0, const int (&image)[2],
                                                  uint64_t policy, const Params& p) {
        const int j0 = row0 / K;  // row0 is a multiple of K (planner)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int w0 = (col0[k] / 124) * L::kU8Words;
#pragma unroll
            for (int r = 0; r < K; ++r)
                tma_load_3d(static_cast<unsigned char*>(smem) + (k * K + r) * kBoxStride, tmap, bar,
                            (r * p.pitch_words + w0) & ~3, j0, image[k], policy);
        }
    }

    __device__ __forceinline__ void begin_tile(const int (&col0)[2], int, const int (&)[2]) {
        const int wa = (col0[0] / 124) * L::kU8Words, wb = (col0[1] / 124) * L::kU8Words;
#pragma unroll
        for (int r = 0; r < K; ++r) {
            skip_a[r] = (r * pw + wa) & 3;
            skip_b[r] = (r * pw + wb) & 3;
        }
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[2][4]) {
        constexpr int cls = R % K, gr = R / K;
        const uint32_t* wa =
            reinterpret_cast<const uint32_t*>(stage + cls * kBoxStride) + gr * kWords + skip_a[cls] + 3 * lane;
        const uint32_t* wb =
            reinterpret_cast<const uint32_t*>(stage + (K + cls) * kBoxStride) + gr * kWords + skip_b[cls] + 3 * lane;
        const uint32_t a[3] = {wa[0], wa[1], wa[2]};
        const uint32_t b[3] = {wb[0], wb[1], wb[2]};
        float2 gown[4];
        gray4_u8x2<EXACT>(a, b, gown[0], gown[1], gown[2], gown[3]);
        core.template step<R, NoHalo, true>(gown, lane, NoHalo{}, out);
    }
};

}  // namespace harris
