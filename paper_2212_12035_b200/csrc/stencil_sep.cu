// stencil_sep.cu — separable 3x3 stencil on the strip engine (SURVEY.md §8(f)
// row 3): out[y][x] = sum_i sum_j wv[i] wh[j] in[y+i][x+j] on one f32 plane,
// valid region (n+2) x (m+2) -> n x m.  This is the reference package's own
// stencil workload, the binomial filter weightsV = weightsH = [1,2,1]
// (evalref.py:112-115; rewrite goal PAPER.md:3935-4016, binomial.rules:26-27),
// evaluated in the goal's *separated* order: a vertical 3-tap per column, then a
// horizontal 3-tap over the column results.
//
// Each lane owns 4 output columns; it reads its float4 plus the next 2 columns of
// the TMA box (so no shuffles and no divergent halo branch), keeps the last 3
// input rows of those 6 columns in registers (slot = row % 3) and emits one
// float4 per row.  EXACT: every product/sum rounded in listing order (bit-exact
// with oracle/stencil_oracle.c); FAST: FMA chains.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "harris_common.cuh"
#include "harris_internal.h"
#include "stencil_sep.cuh"
#include "strip_pipeline.cuh"

namespace harris {

// configs (warps, stages, rows/stage, min CTAs/SM); HARRIS_SEP_CONFIG selects one
template <int CFG>
struct SepCfg;
template <>
struct SepCfg<0> {
    static constexpr int NW = 8, NS = 8, CH = 6, MINB = 1;
};
template <>
struct SepCfg<1> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 2;
};
template <>
struct SepCfg<2> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 1;
};
// 3 (default for 16-byte aligned outputs): TMA-store outputs, 8 warps x 6 stages + 2 output
// staging buffers per warp (202 KB)
template <>
struct SepCfg<3> {
    static constexpr int NW = 8, NS = 6, CH = 6, MINB = 1;
    static constexpr bool TS = true;
};
// 4-8: pipeline-shape sweep (warps x stages x rows per stage), register stores
template <>
struct SepCfg<4> {
    static constexpr int NW = 6, NS = 10, CH = 6, MINB = 1;
};
template <>
struct SepCfg<5> {
    static constexpr int NW = 4, NS = 16, CH = 6, MINB = 1;
};
template <>
struct SepCfg<6> {
    static constexpr int NW = 16, NS = 4, CH = 6, MINB = 1;
};
template <>
struct SepCfg<7> {
    static constexpr int NW = 8, NS = 4, CH = 12, MINB = 1;
};
template <>
struct SepCfg<8> {
    static constexpr int NW = 12, NS = 5, CH = 6, MINB = 1;
};
template <int CFG, class = void>
struct SepTs : std::false_type {};
template <int CFG>
struct SepTs<CFG, std::void_t<decltype(SepCfg<CFG>::TS)>> : std::integral_constant<bool, SepCfg<CFG>::TS> {};

const TmaConfig kSepConfigs[kNumSepConfigs] = {{8, 8, 6}, {8, 4, 6}, {8, 4, 6}, {8, 6, 6}, {6, 10, 6},
                                               {4, 16, 6}, {16, 4, 6}, {8, 4, 12}, {12, 5, 6}};

template <int CFG, bool EXACT>
using SepOpOf = std::conditional_t<SepTs<CFG>::value, Sep3x3TsOp<EXACT, SepCfg<CFG>::CH>,
                                   Sep3x3Op<EXACT, SepCfg<CFG>::CH>>;

template <int CFG, bool EXACT>
static constexpr auto sep_kernel() {
    using C = SepCfg<CFG>;
    return strip_kernel<SepOpOf<CFG, EXACT>, C::NW, C::NS, C::MINB>;
}

template <int CFG>
static constexpr size_t sep_smem() {
    using C = SepCfg<CFG>;
    return StripShape<C::NW, C::NS, SepOpOf<CFG, false>>::kSmemBytes;
}
static_assert(sep_smem<3>() <= 227 * 1024 && sep_smem<4>() <= 227 * 1024 && sep_smem<5>() <= 227 * 1024 &&
                  sep_smem<6>() <= 227 * 1024 && sep_smem<7>() <= 227 * 1024 && sep_smem<8>() <= 227 * 1024,
              "stencil smem");

template <int CFG>
static cudaError_t sep_configure_one(int* ctas_per_sm) {
    using C = SepCfg<CFG>;
    cudaError_t e = cudaFuncSetAttribute(sep_kernel<CFG, false>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sep_smem<CFG>()));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sep_kernel<CFG, true>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sep_smem<CFG>()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, sep_kernel<CFG, false>(), C::NW * 32,
                                                          sep_smem<CFG>());
    return e;
}

cudaError_t sep_configure(int cfg, int* ctas_per_sm) {
    switch (cfg) {
        case 0: return sep_configure_one<0>(ctas_per_sm);
        case 1: return sep_configure_one<1>(ctas_per_sm);
        case 2: return sep_configure_one<2>(ctas_per_sm);
        case 3: return sep_configure_one<3>(ctas_per_sm);
        case 4: return sep_configure_one<4>(ctas_per_sm);
        case 5: return sep_configure_one<5>(ctas_per_sm);
        case 6: return sep_configure_one<6>(ctas_per_sm);
        case 7: return sep_configure_one<7>(ctas_per_sm);
        case 8: return sep_configure_one<8>(ctas_per_sm);
        default: return cudaErrorInvalidValue;
    }
}

template <int CFG, bool EXACT>
static void sep_launch_order(const CUtensorMap& tmap, const CUtensorMap* out_tmap, const TileGeom& tg,
                             int64_t grid, const float* wv, const float* wh, cudaStream_t stream) {
    using C = SepCfg<CFG>;
    using Op = SepOpOf<CFG, EXACT>;
    const dim3 block{unsigned(C::NW * 32)}, gridd{unsigned(grid)};
    typename Sep3x3Op<EXACT, C::CH>::Params base{{wv[0], wv[1], wv[2]}, {wh[0], wh[1], wh[2]}};
    if constexpr (SepTs<CFG>::value) {
        typename Op::Params p;
        p.out = *out_tmap;
        p.base = base;
        launch_strip(sep_kernel<CFG, EXACT>(), gridd, block, sep_smem<CFG>(), stream, tg.pdl, tmap, tg, p);
    } else {
        (void)out_tmap;
        launch_strip(sep_kernel<CFG, EXACT>(), gridd, block, sep_smem<CFG>(), stream, tg.pdl, tmap, tg, base);
    }
}

template <int CFG>
static cudaError_t sep_launch_one(bool exact, const CUtensorMap& tmap, const CUtensorMap* out_tmap,
                                  const TileGeom& tg, int64_t grid, const float* wv, const float* wh,
                                  cudaStream_t stream) {
    if (SepTs<CFG>::value && !out_tmap) return cudaErrorInvalidValue;
    if (exact)
        sep_launch_order<CFG, true>(tmap, out_tmap, tg, grid, wv, wh, stream);
    else
        sep_launch_order<CFG, false>(tmap, out_tmap, tg, grid, wv, wh, stream);
    return cudaGetLastError();
}

bool sep_config_tma_store(int cfg) { return cfg == 3; }

cudaError_t launch_tma_sep(int cfg, bool exact, const CUtensorMap& tmap, const CUtensorMap* out_tmap,
                           const TileGeom& tg, int64_t grid, const float* wv, const float* wh, cudaStream_t stream) {
    switch (cfg) {
        case 0: return sep_launch_one<0>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 1: return sep_launch_one<1>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 2: return sep_launch_one<2>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 3: return sep_launch_one<3>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 4: return sep_launch_one<4>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 5: return sep_launch_one<5>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 6: return sep_launch_one<6>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 7: return sep_launch_one<7>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        case 8: return sep_launch_one<8>(exact, tmap, out_tmap, tg, grid, wv, wh, stream);
        default: return cudaErrorInvalidValue;
    }
}

// generic fallback: one thread per output pixel, same two orders
template <bool EXACT>
__global__ void sep_generic_kernel(const float* __restrict__ in, int64_t in_pitch, int64_t in_image_stride,
                                   float* __restrict__ out, int64_t out_pitch, int64_t out_image_stride, int64_t n,
                                   int64_t m, int64_t batch, float wv0, float wv1, float wv2, float wh0, float wh1,
                                   float wh2) {
    const int64_t total = batch * n * m;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = e % m, yb = e / m, y = yb % n, b = yb / n;
        const float* p = in + b * in_image_stride + y * in_pitch + x;
        float v[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float r0 = __ldg(p + j), r1 = __ldg(p + in_pitch + j), r2 = __ldg(p + 2 * in_pitch + j);
            if (EXACT) {
                float t = __fadd_rn(0.0f, __fmul_rn(wv0, r0));
                t = __fadd_rn(t, __fmul_rn(wv1, r1));
                v[j] = __fadd_rn(t, __fmul_rn(wv2, r2));
            } else {
                v[j] = fmaf(wv2, r2, fmaf(wv1, r1, wv0 * r0));
            }
        }
        float o;
        if (EXACT) {
            float t = __fadd_rn(0.0f, __fmul_rn(wh0, v[0]));
            t = __fadd_rn(t, __fmul_rn(wh1, v[1]));
            o = __fadd_rn(t, __fmul_rn(wh2, v[2]));
        } else {
            o = fmaf(wh2, v[2], fmaf(wh1, v[1], wh0 * v[0]));
        }
        out[b * out_image_stride + y * out_pitch + x] = o;
    }
}

cudaError_t launch_generic_sep(bool exact, const float* in, int64_t in_pitch, int64_t in_image_stride, float* out,
                               int64_t out_pitch, int64_t out_image_stride, int64_t n, int64_t m, int64_t batch,
                               const float* wv, const float* wh, int num_sms, cudaStream_t stream) {
    const int64_t total = batch * n * m;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = int64_t(num_sms) * 16;
    if (blocks > cap) blocks = cap;
    if (exact)
        sep_generic_kernel<true><<<unsigned(blocks), 256, 0, stream>>>(in, in_pitch, in_image_stride, out, out_pitch,
                                                                       out_image_stride, n, m, batch, wv[0], wv[1],
                                                                       wv[2], wh[0], wh[1], wh[2]);
    else
        sep_generic_kernel<false><<<unsigned(blocks), 256, 0, stream>>>(in, in_pitch, in_image_stride, out,
                                                                        out_pitch, out_image_stride, n, m, batch,
                                                                        wv[0], wv[1], wv[2], wh[0], wh[1], wh[2]);
    return cudaGetLastError();
}

}  // namespace harris
