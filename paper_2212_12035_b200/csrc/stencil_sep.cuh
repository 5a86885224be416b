// stencil_sep.cuh — the separable 3x3 stencil as a strip-pipeline op (SURVEY.md §8(f)
// row 3; the reference's binomial goal), shared by the TMA kernel
// (stencil_sep.cu) and the cp.async kernel for planes TMA cannot describe (harris_ldg.cu).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "harris_common.cuh"
#include "harris_internal.h"

namespace harris {

template <bool EXACT, int CH>
struct Sep3x3Op {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    static constexpr int kGroups = 1;
    static constexpr int kPlanes = 1;
    static constexpr int kStripCols = kWarpCols;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kHaloRows = 2;
    static constexpr bool kTwoStoreVariants = true;  // measured +5 % on unaligned planes
    static constexpr bool kRealignStores = true;     // 8-byte aligned output rows: 16-byte stores anyway
    static constexpr uint32_t kTxBytes = uint32_t(CH) * kBoxCols * 4u;
    static constexpr uint32_t kStageBytes = (kTxBytes + 127u) / 128u * 128u;
    struct Params {
        float wv[3], wh[3];
    };
    float wv0, wv1, wv2, wh0, wh1, wh2;
    float X[3][6];

    __device__ __forceinline__ explicit Sep3x3Op(const Params& p)
        : wv0(p.wv[0]), wv1(p.wv[1]), wv2(p.wv[2]), wh0(p.wh[0]), wh1(p.wh[1]), wh2(p.wh[2]) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 6; ++k) X[a][k] = 0.f;
    }

    __device__ __forceinline__ static void load(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                const int (&col0)[1], int row0, const int (&image)[1],
                                                uint64_t policy) {
        tma_load_3d(smem, tmap, bar, col0[0], row0, image[0], policy);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out4)[1][4]) {
        const float* rp = reinterpret_cast<const float*>(stage) + R * kBoxCols + lane * 4;
        const float4 a = lds128(rp);
        const float2 b = *reinterpret_cast<const float2*>(rp + 4);
        const float x[6] = {a.x, a.y, a.z, a.w, b.x, b.y};
        compute<R>(x, out4[0]);
    }

    // input row R (6 columns of this lane: its 4 + the 2-column halo) -> 4 outputs
    template <int R>
    __device__ __forceinline__ void compute(const float (&x)[6], float (&out)[4]) {
        constexpr int s2 = R % 3, s0 = (R + 1) % 3, s1 = (R + 2) % 3;
#pragma unroll
        for (int j = 0; j < 6; ++j) X[s2][j] = x[j];
        float v[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            if constexpr (EXACT) {
                float t = __fadd_rn(0.0f, __fmul_rn(wv0, X[s0][j]));
                t = __fadd_rn(t, __fmul_rn(wv1, X[s1][j]));
                v[j] = __fadd_rn(t, __fmul_rn(wv2, X[s2][j]));
            } else {
                v[j] = fmaf(wv2, X[s2][j], fmaf(wv1, X[s1][j], wv0 * X[s0][j]));
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if constexpr (EXACT) {
                float t = __fadd_rn(0.0f, __fmul_rn(wh0, v[k]));
                t = __fadd_rn(t, __fmul_rn(wh1, v[k + 1]));
                out[k] = __fadd_rn(t, __fmul_rn(wh2, v[k + 2]));
            } else {
                out[k] = fmaf(wh2, v[k + 2], fmaf(wh1, v[k + 1], wh0 * v[k]));
            }
        }
    }
};

// The same stencil with TMA-store outputs (strip engine kTmaStore): a lane writes its 4
// outputs per row to the warp's staging buffer, lane 0 stores 128 x 2-row boxes through the
// output tensor map.  The 1:1 read/write mix of this op leaves the register-store version
// short of the copy ceiling (outstanding writes per SM with 8 warps); bulk stores move the
// write stream to the TMA unit.  Needs 16-byte aligned output rows (tensor-map strides).
template <bool EXACT, int CH>
struct Sep3x3TsOp : Sep3x3Op<EXACT, CH> {
    using Base = Sep3x3Op<EXACT, CH>;
    static constexpr bool kTmaStore = true;
    static constexpr uint32_t kOutStageBytes = uint32_t(CH) * kWarpCols * 4u;
    struct Params {
        CUtensorMap out;  // {m, n, batch} f32, box {128, 2, 1}
        typename Base::Params base;
    };
    __device__ __forceinline__ explicit Sep3x3TsOp(const Params& p) : Base(p.base) {}
    __device__ __forceinline__ static const void* out_tmap(const Params& p) { return &p.out; }
};

}  // namespace harris
