// harris_tma.cu — K1: the fused Harris kernel for sm_100a.
//
// One kernel runs all five stages of the thesis pipeline (gray -> Sobel Ix/Iy ->
// products -> 3x3 box sums -> coarsity); no intermediate
// touches HBM.  The six thesis optimisations map to:
//
//  * operator fusion        — everything below happens in registers; the only
//                             global traffic is 12 B/px in and 4 B/px out.
//  * multithreading         — persistent 2-D strip grid: a *tile* is one
//                             128-column warp strip x `band_rows` output rows of
//                             one image; warps stride over tiles (grid = SMs x
//                             resident CTAs).  Bands re-read a 4-row halo.
//  * vectorisation          — each lane owns 4 adjacent columns: one float4 per
//                             channel per row from shared memory, one 16-byte
//                             streaming store per output row.
//  * TMA staging            — each warp owns an NS-stage ring in shared memory;
//                             lane 0 issues one 4-D cp.async.bulk.tensor box per
//                             stage ({132 cols, CH rows, 3 channels, 1 image},
//                             OOB zero-filled) completing on a per-stage
//                             mbarrier.  The producer cursor runs NS stages ahead
//                             of the consumer and continues across tiles, so the
//                             pipeline never drains between tiles.
//  * circular buffering +   — the warp marches down its strip one input row at a
//    register rotation        time, keeping only the 3-row windows the stencils
//                             need (Sobel partials, then box partials) in
//                             registers, rotated by renaming: CH is a multiple of
//                             3 and the row loop is fully unrolled, so row i
//                             always lives in slot i%3 (cbuf+rrot,
//                             PAPER.md:4814-4815, 4927-4929).
//  * convolution separation — FAST mode: vertical/horizontal separated Sobel and
//                             box sums.
//  * halo exchange          — the 4 columns right of a lane's float4 come from
//                             lane+1 via __shfl_down_sync; lane 31 reads the
//                             4-column halo of the TMA box from shared memory.
//
// The engine itself (tiles, TMA ring, mbarriers, stores) is strip_pipeline.cuh;
// the per-row arithmetic is HarrisF32Op in harris_ops.cuh.
//
// EXACT mode keeps the same schedule but evaluates the Appendix-B op order with
// non-contracted intrinsics, so its output is bit-identical to the C oracle.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "harris_common.cuh"
#include "harris_internal.h"
#include "harris_ops.cuh"
#include "harris_ops2.cuh"
#include "strip_pipeline.cuh"

namespace harris {

// (warps per CTA, stages per warp, rows per stage, min CTAs per SM); index 0 is the
// default, HARRIS_TMA_CONFIG selects another (tools/probe_perf.py sweeps them)
template <int CFG>
struct F32Cfg;
// scalar single-strip core
template <> struct F32Cfg<0> { static constexpr int NW = 8, NS = 3, CH = 3, MINB = 1, G = 1; };
template <> struct F32Cfg<1> { static constexpr int NW = 8, NS = 2, CH = 3, MINB = 2, G = 1; };
template <> struct F32Cfg<2> { static constexpr int NW = 4, NS = 3, CH = 3, MINB = 3, G = 1; };
template <> struct F32Cfg<3> { static constexpr int NW = 4, NS = 4, CH = 3, MINB = 1, G = 1; };
template <> struct F32Cfg<4> { static constexpr int NW = 4, NS = 3, CH = 6, MINB = 1, G = 1; };
// packed FP32x2 dual-strip core (harris_ops2.cuh)
template <> struct F32Cfg<5> { static constexpr int NW = 6, NS = 3, CH = 3, MINB = 1, G = 2; };
template <> struct F32Cfg<6> { static constexpr int NW = 8, NS = 2, CH = 3, MINB = 1, G = 2; };
template <> struct F32Cfg<7> { static constexpr int NW = 4, NS = 4, CH = 3, MINB = 1, G = 2; };
// scalar core, deep ring (small images: more of each short tile in flight)
template <> struct F32Cfg<8> { static constexpr int NW = 8, NS = 4, CH = 3, MINB = 1, G = 1; };
// 124-column lane-halo strips (harris_common.cuh Strip<124>): no lane-31 halo branch
template <> struct F32Cfg<9> { static constexpr int NW = 8, NS = 2, CH = 3, MINB = 1, G = 2, SC = 124; };
template <> struct F32Cfg<10> { static constexpr int NW = 8, NS = 3, CH = 3, MINB = 1, G = 1, SC = 124; };

template <class C, class = void>
struct StripColsOf : std::integral_constant<int, 128> {};
template <class C>
struct StripColsOf<C, std::void_t<decltype(C::SC)>> : std::integral_constant<int, C::SC> {};

template <int CFG, bool EXACT, int WIN = 0>
using F32OpOf = std::conditional_t<F32Cfg<CFG>::G == 2,
                                   HarrisF32x2Op<EXACT, F32Cfg<CFG>::CH, StripColsOf<F32Cfg<CFG>>::value, WIN>,
                                   HarrisF32Op<EXACT, F32Cfg<CFG>::CH, StripColsOf<F32Cfg<CFG>>::value, WIN>>;

#define HARRIS_CFG_ROW(k) {F32Cfg<k>::NW, F32Cfg<k>::NS, F32Cfg<k>::CH, F32Cfg<k>::G, StripColsOf<F32Cfg<k>>::value}
const TmaConfig kTmaConfigs[kNumTmaConfigs] = {
    HARRIS_CFG_ROW(0), HARRIS_CFG_ROW(1), HARRIS_CFG_ROW(2), HARRIS_CFG_ROW(3), HARRIS_CFG_ROW(4),
    HARRIS_CFG_ROW(5), HARRIS_CFG_ROW(6), HARRIS_CFG_ROW(7), HARRIS_CFG_ROW(8), HARRIS_CFG_ROW(9),
    HARRIS_CFG_ROW(10),
};
#undef HARRIS_CFG_ROW

template <int CFG, bool EXACT, int WIN = 0>
static constexpr auto f32_kernel() {
    using C = F32Cfg<CFG>;
    return strip_kernel<F32OpOf<CFG, EXACT, WIN>, C::NW, C::NS, C::MINB>;
}

template <int CFG>
static constexpr size_t f32_smem() {
    using C = F32Cfg<CFG>;
    return StripShape<C::NW, C::NS, F32OpOf<CFG, false>>::kSmemBytes;
}

constexpr size_t kMaxDynSmem = 227 * 1024;  // sm_100 opt-in maximum per block

template <int CFG, int WIN = 0>
static cudaError_t configure_one() {
    static_assert(f32_smem<CFG>() <= kMaxDynSmem, "TMA config exceeds 227 KB of shared memory");
    cudaError_t e = cudaFuncSetAttribute(f32_kernel<CFG, false, WIN>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(f32_smem<CFG>()));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(f32_kernel<CFG, true, WIN>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(f32_smem<CFG>()));
}

template <int CFG, int WIN = 0>
static cudaError_t launch_one(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                              cudaStream_t stream) {
    using C = F32Cfg<CFG>;
    const dim3 block{unsigned(C::NW * 32)}, gridd{unsigned(grid)};
    if (exact) {
        const typename F32OpOf<CFG, true, WIN>::Params p{tg.kappa};
        launch_strip(f32_kernel<CFG, true, WIN>(), gridd, block, f32_smem<CFG>(), stream, tg.pdl, tmap, tg, p);
    } else {
        const typename F32OpOf<CFG, false, WIN>::Params p{tg.kappa};
        launch_strip(f32_kernel<CFG, false, WIN>(), gridd, block, f32_smem<CFG>(), stream, tg.pdl, tmap, tg, p);
    }
    return cudaGetLastError();
}

// ---- Harris with the binomial window (WIN = 1): the default long-tile config (6, packed
// dual-strip core) and the short-tile config (0, scalar core) only
bool tma_window_config(int cfg) { return cfg == 0 || cfg == 6; }

cudaError_t tma_window_configure() {
    cudaError_t e = configure_one<0, 1>();
    return e == cudaSuccess ? configure_one<6, 1>() : e;
}

cudaError_t tma_window_occupancy(int cfg, int* ctas_per_sm) {
    if (cfg == 0)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, f32_kernel<0, false, 1>(),
                                                             F32Cfg<0>::NW * 32, f32_smem<0>());
    if (cfg == 6)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, f32_kernel<6, false, 1>(),
                                                             F32Cfg<6>::NW * 32, f32_smem<6>());
    return cudaErrorInvalidValue;
}

cudaError_t launch_tma_window(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                              cudaStream_t stream) {
    if (cfg == 0) return launch_one<0, 1>(exact, tmap, tg, grid, stream);
    if (cfg == 6) return launch_one<6, 1>(exact, tmap, tg, grid, stream);
    return cudaErrorInvalidValue;
}

template <int CFG>
static cudaError_t occupancy_one(int* n) {
    using C = F32Cfg<CFG>;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, f32_kernel<CFG, false>(), C::NW * 32, f32_smem<CFG>());
}

#define HARRIS_F32_SWITCH(EXPR_T)       \
    switch (cfg) {                      \
        case 0: return EXPR_T(0);       \
        case 1: return EXPR_T(1);       \
        case 2: return EXPR_T(2);       \
        case 3: return EXPR_T(3);       \
        case 4: return EXPR_T(4);       \
        case 5: return EXPR_T(5);       \
        case 6: return EXPR_T(6);       \
        case 7: return EXPR_T(7);       \
        case 8: return EXPR_T(8);       \
        case 9: return EXPR_T(9);       \
        case 10: return EXPR_T(10);     \
        default: break;                 \
    }

size_t tma_smem_bytes(int cfg) {
#define E(k) f32_smem<k>()
    HARRIS_F32_SWITCH(E)
#undef E
    return 0;
}

cudaError_t tma_configure(int cfg) {
#define E(k) configure_one<k>()
    HARRIS_F32_SWITCH(E)
#undef E
    return cudaErrorInvalidValue;
}

cudaError_t tma_occupancy(int cfg, int* ctas_per_sm) {
#define E(k) occupancy_one<k>(ctas_per_sm)
    HARRIS_F32_SWITCH(E)
#undef E
    return cudaErrorInvalidValue;
}

cudaError_t launch_tma(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                       cudaStream_t stream) {
#define E(k) launch_one<k>(exact, tmap, tg, grid, stream)
    HARRIS_F32_SWITCH(E)
#undef E
    return cudaErrorInvalidValue;
}

// ---- pair-row TMA kernel (row pitch = 2 mod 4 floats, HarrisF32PairRowOp) ----
constexpr int kPairNW = 8, kPairNS = 2;
const TmaConfig kPairConfig = {kPairNW, kPairNS, 6, 1, 124};

template <bool EXACT>
static constexpr auto pair_kernel() {
    return strip_kernel<HarrisF32PairRowOp<EXACT>, kPairNW, kPairNS, 1>;
}
static constexpr size_t pair_smem() { return StripShape<kPairNW, kPairNS, HarrisF32PairRowOp<false>>::kSmemBytes; }
static_assert(pair_smem() <= 227 * 1024, "pair-row config exceeds 227 KB of shared memory");

cudaError_t pair_configure(int* ctas_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(pair_kernel<false>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(pair_smem()));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(pair_kernel<true>(), cudaFuncAttributeMaxDynamicSharedMemorySize, int(pair_smem()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, pair_kernel<false>(), kPairNW * 32,
                                                          pair_smem());
    return e;
}

cudaError_t launch_tma_pair(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid, int32_t pitch,
                            cudaStream_t stream) {
    const dim3 block{unsigned(kPairNW * 32)}, gridd{unsigned(grid)};
    if (exact)
        launch_strip(pair_kernel<true>(), gridd, block, pair_smem(), stream, tg.pdl, tmap, tg,
                                                                  typename HarrisF32PairRowOp<true>::Params{tg.kappa, pitch});
    else
        launch_strip(pair_kernel<false>(), gridd, block, pair_smem(), stream, tg.pdl, tmap, tg, typename HarrisF32PairRowOp<false>::Params{tg.kappa, pitch});
    return cudaGetLastError();
}

// ---- quad-row TMA kernel (odd row pitch, HarrisF32QuadRowOp): 12-row stages, 4 warps (one per SMSP) ----
#ifndef HARRIS_QUAD_NW
#define HARRIS_QUAD_NW 4
#define HARRIS_QUAD_NS 2
#endif
constexpr int kQuadNW = HARRIS_QUAD_NW, kQuadNS = HARRIS_QUAD_NS;
const TmaConfig kQuadConfig = {kQuadNW, kQuadNS, 12, 1, 124};

template <bool EXACT>
static constexpr auto quad_kernel() {
    return strip_kernel<HarrisF32QuadRowOp<EXACT>, kQuadNW, kQuadNS, 1>;
}
static constexpr size_t quad_smem() { return StripShape<kQuadNW, kQuadNS, HarrisF32QuadRowOp<false>>::kSmemBytes; }
static_assert(quad_smem() <= 227 * 1024, "quad-row config exceeds 227 KB of shared memory");

cudaError_t quad_configure(int* ctas_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(quad_kernel<false>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(quad_smem()));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(quad_kernel<true>(), cudaFuncAttributeMaxDynamicSharedMemorySize, int(quad_smem()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, quad_kernel<false>(), kQuadNW * 32,
                                                          quad_smem());
    return e;
}

cudaError_t launch_tma_quad(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid, int32_t pitch,
                            cudaStream_t stream) {
    const dim3 block{unsigned(kQuadNW * 32)}, gridd{unsigned(grid)};
    if (exact)
        launch_strip(quad_kernel<true>(), gridd, block, quad_smem(), stream, tg.pdl, tmap, tg,
                                                                  typename HarrisF32QuadRowOp<true>::Params{tg.kappa, pitch});
    else
        launch_strip(quad_kernel<false>(), gridd, block, quad_smem(), stream, tg.pdl, tmap, tg, typename HarrisF32QuadRowOp<false>::Params{tg.kappa, pitch});
    return cudaGetLastError();
}

}  // namespace harris
