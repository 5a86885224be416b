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
// EXACT mode keeps the same schedule but evaluates the Appendix-B op order with
// non-contracted intrinsics, so its output is bit-identical to the C oracle.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "harris_common.cuh"
#include "harris_internal.h"

namespace harris {

const TmaConfig kTmaConfigs[kNumTmaConfigs] = {
    {8, 3, 3},  // 0: default, 117 KB smem / CTA, 1 CTA (8 warps) per SM
    {2, 4, 3},  // 1
    {4, 3, 6},  // 2
    {4, 4, 3},  // 3
};

template <int NW, int NS, int CH>
struct TmaShape {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    static constexpr int kStageFloats = ((3 * CH * kBoxCols + 31) / 32) * 32;  // 128-B aligned stages
    static constexpr uint32_t kTxBytes = 3u * CH * kBoxCols * 4u;              // bytes one box delivers
    static constexpr size_t kSmemBytes = size_t(NW) * NS * kStageFloats * 4 + size_t(NW) * NS * 8 + 128;
};

struct TileCoord {
    int b, band, cs;
};

__device__ __forceinline__ TileCoord decode_tile(int64_t t, const TileGeom& g) {
    TileCoord c;
    int64_t q = t / g.colsegs;
    c.cs = int(t - q * g.colsegs);
    int64_t b = q / g.bands;
    c.band = int(q - b * g.bands);
    c.b = int(b);
    return c;
}

__device__ __forceinline__ int band_rows_out(int band, const TileGeom& g) {
    int r0 = band * g.band_rows;
    int r = g.n - r0;
    return r < g.band_rows ? r : g.band_rows;
}

__device__ __forceinline__ void hsum4(const float (&p)[6], float& o0, float& o1, float& o2, float& o3) {
    const float q1 = p[1] + p[2], q3 = p[3] + p[4];
    o0 = p[0] + q1;
    o1 = q1 + p[3];
    o2 = p[2] + q3;
    o3 = q3 + p[5];
}

template <bool EXACT, int NW, int NS, int CH>
__global__ void __launch_bounds__(NW * 32, 1)
    harris_tma_kernel(const __grid_constant__ CUtensorMap tmap, const TileGeom g) {
    using S = TmaShape<NW, NS, CH>;
    extern __shared__ unsigned char smem_raw[];
    float* base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    float* ring = base + warp * NS * S::kStageFloats;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + NW * NS * S::kStageFloats) + warp * NS;

    const int64_t GW = int64_t(gridDim.x) * NW;
    const int64_t gw = int64_t(blockIdx.x) * NW + warp;
    if (gw >= g.tiles) return;  // warps are independent: no CTA-wide barrier below

    if (lane == 0) {
        prefetch_tmap(&tmap);
#pragma unroll
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncwarp();
    const uint64_t policy = l2_policy(g.l2_policy);

    // ---- producer cursor (warp-uniform; lane 0 issues) ----
    int64_t pt = gw;
    int pc = 0;
    int pn = (band_rows_out(decode_tile(pt, g).band, g) + 4 + CH - 1) / CH;
    auto issue = [&](int s) {
        if (pt < g.tiles) {
            if (lane == 0) {
                TileCoord c = decode_tile(pt, g);
                mbar_arrive_expect_tx(&bars[s], S::kTxBytes);
                tma_load_4d(ring + s * S::kStageFloats, &tmap, &bars[s], c.cs * kWarpCols,
                            c.band * g.band_rows + pc * CH, 0, c.b, policy);
            }
            if (++pc == pn) {
                pc = 0;
                pt += GW;
                if (pt < g.tiles) pn = (band_rows_out(decode_tile(pt, g).band, g) + 4 + CH - 1) / CH;
            }
        }
    };
#pragma unroll
    for (int s = 0; s < NS; ++s) issue(s);

    // ---- consumer: rolling 3-row windows, slot = row % 3 ----
    // FAST: D = horizontal diff g[k+2]-g[k], Hs = horizontal smooth g[k]+2g[k+1]+g[k+2]
    //       (6 Sobel columns), HB = horizontal 3-sums of the products (3 x 4 columns).
    // EXACT: G3 = gray rows (8 columns), P = product rows (3 x 6 columns).
    float D[3][6], Hs[3][6], HB[3][12];
    float G3[3][8], P[3][18];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int k = 0; k < 6; ++k) D[a][k] = Hs[a][k] = 0.f;
#pragma unroll
        for (int k = 0; k < 12; ++k) HB[a][k] = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) G3[a][k] = 0.f;
#pragma unroll
        for (int k = 0; k < 18; ++k) P[a][k] = 0.f;
    }
    const float WX[9] = {-kSobA, 0.f, kSobA, -kSobB, 0.f, kSobB, -kSobA, 0.f, kSobA};
    const float WY[9] = {-kSobA, -kSobB, -kSobA, 0.f, 0.f, 0.f, kSobA, kSobB, kSobA};
    const float kappa = g.kappa;

    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = gw; t < g.tiles; t += GW) {
        const TileCoord tc = decode_tile(t, g);
        const int rows_out = band_rows_out(tc.band, g);
        const int nch = (rows_out + 4 + CH - 1) / CH;
        const int col0 = tc.cs * kWarpCols + lane * kColsPerLane;
        const bool col_ok = col0 < g.m;
        float* orow = g.out + int64_t(tc.b) * g.out_image_stride +
                      int64_t(tc.band) * g.band_rows * g.out_pitch + col0;

        for (int c = 0; c < nch; ++c) {
            mbar_wait(&bars[stage], phase);
            const float* sm = ring + stage * S::kStageFloats;
#pragma unroll
            for (int r = 0; r < CH; ++r) {
                const int i = c * CH + r;           // input row within the tile
                const int s2 = r % 3;               // slot of row i
                const int s0 = (r + 1) % 3;         // slot of row i-2
                const int s1 = (r + 2) % 3;         // slot of row i-1
                const float* pr = sm + (0 * CH + r) * kBoxCols;
                const float* pg = sm + (1 * CH + r) * kBoxCols;
                const float* pb = sm + (2 * CH + r) * kBoxCols;
                const float4 R = lds128(pr + lane * 4), Gc = lds128(pg + lane * 4), B = lds128(pb + lane * 4);
                float out4[4];
                if constexpr (!EXACT) {
                    float gr[8];
                    gr[0] = fmaf(kGrayB12, B.x, fmaf(kGrayG12, Gc.x, kGrayR12 * R.x));
                    gr[1] = fmaf(kGrayB12, B.y, fmaf(kGrayG12, Gc.y, kGrayR12 * R.y));
                    gr[2] = fmaf(kGrayB12, B.z, fmaf(kGrayG12, Gc.z, kGrayR12 * R.z));
                    gr[3] = fmaf(kGrayB12, B.w, fmaf(kGrayG12, Gc.w, kGrayR12 * R.w));
#pragma unroll
                    for (int k = 0; k < 4; ++k) gr[4 + k] = __shfl_down_sync(0xffffffffu, gr[k], 1);
                    if (lane == 31) {
                        const float4 R2 = lds128(pr + kWarpCols), G2 = lds128(pg + kWarpCols),
                                     B2 = lds128(pb + kWarpCols);
                        gr[4] = fmaf(kGrayB12, B2.x, fmaf(kGrayG12, G2.x, kGrayR12 * R2.x));
                        gr[5] = fmaf(kGrayB12, B2.y, fmaf(kGrayG12, G2.y, kGrayR12 * R2.y));
                        gr[6] = fmaf(kGrayB12, B2.z, fmaf(kGrayG12, G2.z, kGrayR12 * R2.z));
                        gr[7] = fmaf(kGrayB12, B2.w, fmaf(kGrayG12, G2.w, kGrayR12 * R2.w));
                    }
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        D[s2][k] = gr[k + 2] - gr[k];
                        Hs[s2][k] = fmaf(2.f, gr[k + 1], gr[k]) + gr[k + 2];
                    }
                    float pxx[6], pxy[6], pyy[6];
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        const float ix = fmaf(2.f, D[s1][k], D[s0][k] + D[s2][k]);
                        const float iy = Hs[s2][k] - Hs[s0][k];
                        pxx[k] = ix * ix;
                        pxy[k] = ix * iy;
                        pyy[k] = iy * iy;
                    }
                    // horizontal 3-sums with shared pairs: 6 adds for 4 outputs
                    hsum4(pxx, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
                    hsum4(pxy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
                    hsum4(pyy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float sxx = (HB[s0][0 + j] + HB[s1][0 + j]) + HB[s2][0 + j];
                        const float sxy = (HB[s0][4 + j] + HB[s1][4 + j]) + HB[s2][4 + j];
                        const float syy = (HB[s0][8 + j] + HB[s1][8 + j]) + HB[s2][8 + j];
                        out4[j] = coarsity_fast(sxx, sxy, syy, kappa);
                    }
                } else {
                    G3[s2][0] = gray_exact(R.x, Gc.x, B.x);
                    G3[s2][1] = gray_exact(R.y, Gc.y, B.y);
                    G3[s2][2] = gray_exact(R.z, Gc.z, B.z);
                    G3[s2][3] = gray_exact(R.w, Gc.w, B.w);
#pragma unroll
                    for (int k = 0; k < 4; ++k) G3[s2][4 + k] = __shfl_down_sync(0xffffffffu, G3[s2][k], 1);
                    if (lane == 31) {
                        const float4 R2 = lds128(pr + kWarpCols), G2 = lds128(pg + kWarpCols),
                                     B2 = lds128(pb + kWarpCols);
                        G3[s2][4] = gray_exact(R2.x, G2.x, B2.x);
                        G3[s2][5] = gray_exact(R2.y, G2.y, B2.y);
                        G3[s2][6] = gray_exact(R2.z, G2.z, B2.z);
                        G3[s2][7] = gray_exact(R2.w, G2.w, B2.w);
                    }
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        const float ix = conv9_exact(WX, G3[s0][k], G3[s0][k + 1], G3[s0][k + 2], G3[s1][k],
                                                     G3[s1][k + 1], G3[s1][k + 2], G3[s2][k], G3[s2][k + 1],
                                                     G3[s2][k + 2]);
                        const float iy = conv9_exact(WY, G3[s0][k], G3[s0][k + 1], G3[s0][k + 2], G3[s1][k],
                                                     G3[s1][k + 1], G3[s1][k + 2], G3[s2][k], G3[s2][k + 1],
                                                     G3[s2][k + 2]);
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
                            sq[q] = sum9_exact(P[s0][o], P[s0][o + 1], P[s0][o + 2], P[s1][o], P[s1][o + 1],
                                               P[s1][o + 2], P[s2][o], P[s2][o + 1], P[s2][o + 2]);
                        }
                        out4[j] = coarsity_exact(sq[0], sq[1], sq[2], kappa);
                    }
                }
                if (i >= 4 && i - 4 < rows_out && col_ok) {
                    float* po = orow + int64_t(i - 4) * g.out_pitch;
                    if (g.vec_store && col0 + kColsPerLane <= g.m) {
                        stg128_cs(po, out4[0], out4[1], out4[2], out4[3]);
                    } else {  // unaligned output rows, or the ragged right edge when m % 4 != 0
#pragma unroll
                        for (int k = 0; k < kColsPerLane; ++k)
                            if (col0 + k < g.m) po[k] = out4[k];
                    }
                }
            }
            __syncwarp();  // every lane is done with this stage: refill it
            issue(stage);
            if (++stage == NS) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
}

// ------------------------------------------------------------------ host side
template <int NW, int NS, int CH>
static cudaError_t configure_one() {
    using S = TmaShape<NW, NS, CH>;
    cudaError_t e = cudaFuncSetAttribute(harris_tma_kernel<false, NW, NS, CH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::kSmemBytes));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(harris_tma_kernel<true, NW, NS, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(S::kSmemBytes));
}

template <int NW, int NS, int CH>
static cudaError_t launch_one(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                              cudaStream_t stream) {
    using S = TmaShape<NW, NS, CH>;
    const dim3 block{unsigned(NW * 32)}, gridd{unsigned(grid)};
    if (exact)
        harris_tma_kernel<true, NW, NS, CH><<<gridd, block, S::kSmemBytes, stream>>>(tmap, tg);
    else
        harris_tma_kernel<false, NW, NS, CH><<<gridd, block, S::kSmemBytes, stream>>>(tmap, tg);
    return cudaGetLastError();
}

template <int NW, int NS, int CH>
static cudaError_t occupancy_one(int* n) {
    using S = TmaShape<NW, NS, CH>;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, harris_tma_kernel<false, NW, NS, CH>, NW * 32,
                                                         S::kSmemBytes);
}

size_t tma_smem_bytes(int cfg) {
    switch (cfg) {
        case 0: return TmaShape<8, 3, 3>::kSmemBytes;
        case 1: return TmaShape<2, 4, 3>::kSmemBytes;
        case 2: return TmaShape<4, 3, 6>::kSmemBytes;
        case 3: return TmaShape<4, 4, 3>::kSmemBytes;
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
