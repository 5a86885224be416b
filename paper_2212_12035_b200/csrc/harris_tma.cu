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

#include "harris_common.cuh"
#include "harris_internal.h"
#include "harris_ops.cuh"
#include "strip_pipeline.cuh"

namespace harris {

const TmaConfig kTmaConfigs[kNumTmaConfigs] = {
    {8, 3, 3},  // 0: default, 117 KB smem / CTA, 1 CTA (8 warps) per SM
    {2, 4, 3},  // 1
    {4, 3, 6},  // 2
    {4, 4, 3},  // 3
};

// ------------------------------------------------------------------ host side
template <int NW, int NS, int CH>
static constexpr size_t smem_of() {
    return StripShape<NW, NS, HarrisF32Op<false, CH>>::kSmemBytes;
}

template <int NW, int NS, int CH>
static cudaError_t configure_one() {
    cudaError_t e = cudaFuncSetAttribute(strip_kernel<HarrisF32Op<false, CH>, NW, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_of<NW, NS, CH>()));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(strip_kernel<HarrisF32Op<true, CH>, NW, NS>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_of<NW, NS, CH>()));
}

template <int NW, int NS, int CH>
static cudaError_t launch_one(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                              cudaStream_t stream) {
    const dim3 block{unsigned(NW * 32)}, gridd{unsigned(grid)};
    if (exact) {
        const typename HarrisF32Op<true, CH>::Params p{tg.kappa};
        strip_kernel<HarrisF32Op<true, CH>, NW, NS><<<gridd, block, smem_of<NW, NS, CH>(), stream>>>(tmap, tg, p);
    } else {
        const typename HarrisF32Op<false, CH>::Params p{tg.kappa};
        strip_kernel<HarrisF32Op<false, CH>, NW, NS><<<gridd, block, smem_of<NW, NS, CH>(), stream>>>(tmap, tg, p);
    }
    return cudaGetLastError();
}

template <int NW, int NS, int CH>
static cudaError_t occupancy_one(int* n) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, strip_kernel<HarrisF32Op<false, CH>, NW, NS>, NW * 32,
                                                         smem_of<NW, NS, CH>());
}

size_t tma_smem_bytes(int cfg) {
    switch (cfg) {
        case 0: return smem_of<8, 3, 3>();
        case 1: return smem_of<2, 4, 3>();
        case 2: return smem_of<4, 3, 6>();
        case 3: return smem_of<4, 4, 3>();
        default: return 0;
    }
}

cudaError_t tma_configure(int cfg) {
    switch (cfg) {
        case 0: return configure_one<8, 3, 3>();
        case 1: return configure_one<2, 4, 3>();
        case 2: return configure_one<4, 3, 6>();
        case 3: return configure_one<4, 4, 3>();
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t tma_occupancy(int cfg, int* ctas_per_sm) {
    switch (cfg) {
        case 0: return occupancy_one<8, 3, 3>(ctas_per_sm);
        case 1: return occupancy_one<2, 4, 3>(ctas_per_sm);
        case 2: return occupancy_one<4, 3, 6>(ctas_per_sm);
        case 3: return occupancy_one<4, 4, 3>(ctas_per_sm);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tma(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                       cudaStream_t stream) {
    switch (cfg) {
        case 0: return launch_one<8, 3, 3>(exact, tmap, tg, grid, stream);
        case 1: return launch_one<2, 4, 3>(exact, tmap, tg, grid, stream);
        case 2: return launch_one<4, 3, 6>(exact, tmap, tg, grid, stream);
        case 3: return launch_one<4, 4, 3>(exact, tmap, tg, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace harris
