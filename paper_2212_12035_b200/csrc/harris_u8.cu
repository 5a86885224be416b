// harris_u8.cu — fused Harris on interleaved 8-bit RGB (HWC, e.g. a decoded
// rgb.png): the u8 -> f32 (value/255) conversion is fused
// into the TMA-staged row step, so HBM sees 3 B per
// input pixel instead of 12 and no separate conversion pass exists.  Same strip
// engine (strip_pipeline.cuh) and Harris core (harris_ops.cuh) as the f32 path;
// results equal the f32 path on the planar image u8/255 (bit-for-bit in EXACT
// order).
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

const TmaConfig kU8Configs[kNumU8Configs] = {
    {8, 4, 6, 1},       // 0: scalar core, 2 CTAs (16 warps) per SM (registers capped at 128)
    {8, 4, 6, 1},       // 1: scalar core, 1 CTA per SM
    {8, 3, 3, 1},       // 2: scalar core
    {8, 4, 6, 2},       // 3: packed FP32x2 dual-strip core
    {8, 3, 3, 2},       // 4: packed FP32x2 dual-strip core
    {8, 4, 6, 1, 124},  // 5: as 0, 124-column lane-halo strips (no lane-31 halo branch)
    {8, 4, 6, 2, 124},  // 6: as 3, 124-column lane-halo strips
};

template <int CFG>
struct U8Cfg;
template <>
struct U8Cfg<0> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 2;
};
template <>
struct U8Cfg<1> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 1;
};
template <>
struct U8Cfg<2> {
    static constexpr int NW = 8, NS = 3, CH = 3, MINB = 1;
};
template <>
struct U8Cfg<3> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 1, G = 2;
};
template <>
struct U8Cfg<4> {
    static constexpr int NW = 8, NS = 3, CH = 3, MINB = 1, G = 2;
};
template <>
struct U8Cfg<5> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 2, SC = 124;
};
template <>
struct U8Cfg<6> {
    static constexpr int NW = 8, NS = 4, CH = 6, MINB = 1, G = 2, SC = 124;
};

template <class C, class = void>
struct GroupsOf : std::integral_constant<int, 1> {};
template <class C>
struct GroupsOf<C, std::void_t<decltype(C::G)>> : std::integral_constant<int, C::G> {};

template <class C, class = void>
struct U8StripColsOf : std::integral_constant<int, 128> {};
template <class C>
struct U8StripColsOf<C, std::void_t<decltype(C::SC)>> : std::integral_constant<int, C::SC> {};

template <int CFG, bool EXACT>
using U8OpOf = std::conditional_t<GroupsOf<U8Cfg<CFG>>::value == 2,
                                  HarrisU8x2Op<EXACT, U8Cfg<CFG>::CH, U8StripColsOf<U8Cfg<CFG>>::value>,
                                  HarrisU8Op<EXACT, U8Cfg<CFG>::CH, U8StripColsOf<U8Cfg<CFG>>::value>>;

template <int CFG, bool EXACT>
static constexpr auto u8_kernel() {
    using C = U8Cfg<CFG>;
    return strip_kernel<U8OpOf<CFG, EXACT>, C::NW, C::NS, C::MINB>;
}

template <int CFG>
static constexpr size_t u8_smem() {
    using C = U8Cfg<CFG>;
    return StripShape<C::NW, C::NS, U8OpOf<CFG, false>>::kSmemBytes;
}

template <int CFG>
static cudaError_t u8_configure_one() {
    static_assert(u8_smem<CFG>() <= 227 * 1024, "u8 config exceeds 227 KB of shared memory");
    cudaError_t e = cudaFuncSetAttribute(u8_kernel<CFG, false>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(u8_smem<CFG>()));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(u8_kernel<CFG, true>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(u8_smem<CFG>()));
}

template <int CFG>
static cudaError_t u8_launch_one(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                                 cudaStream_t stream) {
    using C = U8Cfg<CFG>;
    const dim3 block{unsigned(C::NW * 32)}, gridd{unsigned(grid)};
    if (exact) {
        const typename U8OpOf<CFG, true>::Params p{tg.kappa};
        launch_strip(u8_kernel<CFG, true>(), gridd, block, u8_smem<CFG>(), stream, tg.pdl, tmap, tg, p);
    } else {
        const typename U8OpOf<CFG, false>::Params p{tg.kappa};
        launch_strip(u8_kernel<CFG, false>(), gridd, block, u8_smem<CFG>(), stream, tg.pdl, tmap, tg, p);
    }
    return cudaGetLastError();
}

template <int CFG>
static cudaError_t u8_occupancy_one(int* n) {
    using C = U8Cfg<CFG>;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, u8_kernel<CFG, false>(), C::NW * 32, u8_smem<CFG>());
}

size_t u8_smem_bytes(int cfg) {
    switch (cfg) {
        case 0: return u8_smem<0>();
        case 1: return u8_smem<1>();
        case 2: return u8_smem<2>();
        case 3: return u8_smem<3>();
        case 4: return u8_smem<4>();
        case 5: return u8_smem<5>();
        case 6: return u8_smem<6>();
        default: return 0;
    }
}

cudaError_t u8_configure(int cfg) {
    switch (cfg) {
        case 0: return u8_configure_one<0>();
        case 1: return u8_configure_one<1>();
        case 2: return u8_configure_one<2>();
        case 3: return u8_configure_one<3>();
        case 4: return u8_configure_one<4>();
        case 5: return u8_configure_one<5>();
        case 6: return u8_configure_one<6>();
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t u8_occupancy(int cfg, int* ctas_per_sm) {
    switch (cfg) {
        case 0: return u8_occupancy_one<0>(ctas_per_sm);
        case 1: return u8_occupancy_one<1>(ctas_per_sm);
        case 2: return u8_occupancy_one<2>(ctas_per_sm);
        case 3: return u8_occupancy_one<3>(ctas_per_sm);
        case 4: return u8_occupancy_one<4>(ctas_per_sm);
        case 5: return u8_occupancy_one<5>(ctas_per_sm);
        case 6: return u8_occupancy_one<6>(ctas_per_sm);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tma_u8(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                          cudaStream_t stream) {
    switch (cfg) {
        case 0: return u8_launch_one<0>(exact, tmap, tg, grid, stream);
        case 1: return u8_launch_one<1>(exact, tmap, tg, grid, stream);
        case 2: return u8_launch_one<2>(exact, tmap, tg, grid, stream);
        case 3: return u8_launch_one<3>(exact, tmap, tg, grid, stream);
        case 4: return u8_launch_one<4>(exact, tmap, tg, grid, stream);
        case 5: return u8_launch_one<5>(exact, tmap, tg, grid, stream);
        case 6: return u8_launch_one<6>(exact, tmap, tg, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

// ---- row-group TMA kernels for u8 rows TMA cannot step singly (HarrisU8RowGroupOp):
// pairs (pitch = 8 mod 16 bytes, e.g. 1080 px wide) and quads (pitch = 4 mod 8)
const TmaConfig kU8PairConfig = {8, 4, 6, 2, 124};
const TmaConfig kU8QuadConfig = {8, 2, 12, 2, 124};

template <int K>
struct U8GroupCfg {
    static constexpr int NW = 8, NS = K == 2 ? 4 : 2;
};
template <bool EXACT, int K>
static constexpr auto u8_group_kernel() {
    return strip_kernel<HarrisU8RowGroupOp<EXACT, K>, U8GroupCfg<K>::NW, U8GroupCfg<K>::NS, 1>;
}
template <int K>
static constexpr size_t u8_group_smem() {
    return StripShape<U8GroupCfg<K>::NW, U8GroupCfg<K>::NS, HarrisU8RowGroupOp<false, K>>::kSmemBytes;
}
static_assert(u8_group_smem<2>() <= 227 * 1024 && u8_group_smem<4>() <= 227 * 1024, "u8 row-group smem");

template <int K>
static cudaError_t u8_group_configure_one(int* ctas_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(u8_group_kernel<false, K>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(u8_group_smem<K>()));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(u8_group_kernel<true, K>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(u8_group_smem<K>()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, u8_group_kernel<false, K>(),
                                                          U8GroupCfg<K>::NW * 32, u8_group_smem<K>());
    return e;
}

cudaError_t u8_group_configure(int* occ_pair, int* occ_quad) {
    cudaError_t e = u8_group_configure_one<2>(occ_pair);
    return e == cudaSuccess ? u8_group_configure_one<4>(occ_quad) : e;
}

template <bool EXACT, int K>
static void u8_group_launch_one(const CUtensorMap& tmap, const TileGeom& tg, int64_t grid, int32_t pitch_words,
                                cudaStream_t stream) {
    const typename HarrisU8RowGroupOp<EXACT, K>::Params p{tg.kappa, pitch_words};
    launch_strip(u8_group_kernel<EXACT, K>(), unsigned(grid), unsigned(U8GroupCfg<K>::NW * 32), u8_group_smem<K>(), stream, tg.pdl, tmap, tg, p);
}

cudaError_t launch_tma_u8_group(int k, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                                int32_t pitch_words, cudaStream_t stream) {
    if (k == 2)
        exact ? u8_group_launch_one<true, 2>(tmap, tg, grid, pitch_words, stream)
              : u8_group_launch_one<false, 2>(tmap, tg, grid, pitch_words, stream);
    else
        exact ? u8_group_launch_one<true, 4>(tmap, tg, grid, pitch_words, stream)
              : u8_group_launch_one<false, 4>(tmap, tg, grid, pitch_words, stream);
    return cudaGetLastError();
}

}  // namespace harris
