// harris_internal.h — declarations shared between the kernel translation units
// and the C-ABI layer (not part of the public ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>

namespace harris {

// Image geometry of one harris_run_strided call (element strides, not bytes).
struct Geom {
    int64_t n, m, batch;                       // output rows, cols; images
    const float* rgb;
    int64_t in_pitch, in_chan_stride, in_image_stride;
    float* out;
    int64_t out_pitch, out_image_stride;
    float kappa;
    int32_t window = 0;  // 1: binomial window instead of the 3x3 box (generic kernel)
};

// Tile decomposition for the TMA kernel: a tile is one 128-column warp strip of
// `band_rows` output rows of one image.
struct TileGeom {
    int32_t n, m;
    int32_t band_rows, bands, colsegs;  // colsegs: 128-column strips per image
    int32_t batch;
    int32_t l2_policy;  // 0 evict_first, 1 evict_normal, 2 evict_last (default, harris_options)
    int32_t vec_store;  // 2: output rows 16-byte aligned (float4 stores); 1: 8-byte aligned (2 x float2); 0: scalar
    int32_t sync_waves; // 1: CTA barrier at every tile boundary (keeps neighbour strips in step)
    int32_t pdl = 0;    // programmatic dependent launch: 0 off; 1 on (griddepcontrol.wait before the first
                        // global access); 2 on, caller-declared independent of the previous stream work (no wait)
    int64_t tiles;
    int64_t out_pitch, out_image_stride;
    float* out;
    float kappa;
    // completion notification (harris_run_notify): when notify_flag != nullptr, the last
    // CTA to finish stores notify_epoch to *notify_flag (release, system scope) after every
    // CTA's output stores are performed at system scope; notify_counter (device, zeroed)
    // counts finished CTAs and is reset by that last CTA.
    uint32_t* notify_counter = nullptr;
    uint32_t* notify_flag = nullptr;
    uint32_t notify_epoch = 0;
    int64_t out_plane_stride = 0;  // Op::kOutPlanes > 1: elements between output planes
};

// TMA kernel configurations (warps per CTA, pipeline stages per warp, input rows
// per stage).  Index 0 is the default; HARRIS_TMA_CONFIG selects another one.
struct TmaConfig {
    int warps, stages, rows;
    int groups = 1;        // strips per tile (2: packed FP32x2 dual-strip op)
    int strip_cols = 128;  // output columns per strip (124: lane 31 is the halo lane)
};
constexpr int kNumTmaConfigs = 11;
constexpr int kDefaultTmaConfig = 6;  // packed FP32x2 dual-strip core, 8 warps x 2 stages (bench r01)
extern const TmaConfig kTmaConfigs[kNumTmaConfigs];

size_t tma_smem_bytes(int cfg);
cudaError_t tma_configure(int cfg);                                   // smem attribute, once
cudaError_t tma_occupancy(int cfg, int* ctas_per_sm);
cudaError_t launch_tma(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                       cudaStream_t stream);

cudaError_t launch_generic(bool exact, const Geom& g, cudaStream_t stream);

// Harris with the binomial window (HARRIS_FLAG_BINOMIAL_WINDOW): TMA configs 0 and 6
bool tma_window_config(int cfg);
cudaError_t tma_window_configure();
cudaError_t tma_window_occupancy(int cfg, int* ctas_per_sm);
cudaError_t launch_tma_window(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                              cudaStream_t stream);

// pair-row TMA kernel for planar f32 whose row pitch is 2 (mod 4) floats (HarrisF32PairRowOp)
extern const TmaConfig kPairConfig;
cudaError_t pair_configure(int* ctas_per_sm);
cudaError_t launch_tma_pair(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid, int32_t pitch,
                            cudaStream_t stream);
// quad-row TMA kernel for planar f32 with an odd row pitch (HarrisF32QuadRowOp)
extern const TmaConfig kQuadConfig;
cudaError_t quad_configure(int* ctas_per_sm);
cudaError_t launch_tma_quad(bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid, int32_t pitch,
                            cudaStream_t stream);

// cp.async (LDGSTS) warp-strip kernel for f32 inputs TMA cannot describe (row pitch or
// base not 16-byte aligned): same engine and dual-strip core as the TMA path
constexpr int kNumLdgConfigs = 5;
extern const TmaConfig kLdgConfigs[kNumLdgConfigs];
cudaError_t ldg_configure(int cfg, int* ctas_per_sm);
cudaError_t launch_ldg(int cfg, bool exact, const Geom& g, const TileGeom& tg, int64_t grid, cudaStream_t stream);
// interleaved u8 inputs whose byte strides TMA cannot describe (3W % 16 != 0)
extern const TmaConfig kU8LdgConfig;
extern const TmaConfig kU8BulkConfig;
cudaError_t u8_ldg_configure(int* ctas_per_sm, int* bulk_ctas_per_sm);
cudaError_t launch_u8_ldg(bool exact, int chunk, const Geom& g, const TileGeom& tg, int64_t grid,
                          cudaStream_t stream);
// separable stencil planes TMA cannot describe
extern const TmaConfig kSepLdgConfig;
cudaError_t sep_ldg_configure(int* ctas_per_sm);
cudaError_t launch_sep_ldg(bool exact, const float* in, int64_t in_pitch, int64_t in_image_stride, int64_t W,
                           int64_t H, const TileGeom& tg, int64_t grid, const float* wv, const float* wh,
                           cudaStream_t stream);

// interleaved RGB u8 (HWC) input: TMA configs + generic fallback (Geom.rgb is then the
// byte base pointer; in_pitch / in_image_stride are in BYTES, in_chan_stride unused)
constexpr int kNumU8Configs = 7;
// 124-column lane-halo strips: the u8 op is issue-bound and the halo branch was ~17 % of
// its instructions.  Config 6 = the packed dual-strip core in that layout (Sobel sharing,
// producer tile cache): 745.6 k vs 717.8 k MP/s for the scalar core at 16 warps/SM (config 5)
// on configs[4] as u8 (10 launches after 3 warm-ups, 3 alternations)
constexpr int kDefaultU8Config = 6;
extern const TmaConfig kU8Configs[kNumU8Configs];
size_t u8_smem_bytes(int cfg);
cudaError_t u8_configure(int cfg);
cudaError_t u8_occupancy(int cfg, int* ctas_per_sm);
cudaError_t launch_tma_u8(int cfg, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                          cudaStream_t stream);
cudaError_t launch_generic_u8(bool exact, const Geom& g, cudaStream_t stream);
// u8 rows whose pitch is 4, 8 or 12 (mod 16) bytes: TMA over pairs / quads of rows
extern const TmaConfig kU8PairConfig;
extern const TmaConfig kU8QuadConfig;
cudaError_t u8_group_configure(int* occ_pair, int* occ_quad);
cudaError_t launch_tma_u8_group(int k, bool exact, const CUtensorMap& tmap, const TileGeom& tg, int64_t grid,
                                int32_t pitch_words, cudaStream_t stream);

// separable 3x3 stencil on one f32 plane (stencil_sep.cu)
constexpr int kNumSepConfigs = 9;
constexpr int kSepTmaStoreConfig = 3;  // TMA-store epilogue (16-byte aligned outputs with m % 4 == 0)
constexpr int64_t kSepMaxBandRows = 136;  // tile-height cap of the TMA-loaded stencil
extern const TmaConfig kSepConfigs[kNumSepConfigs];
cudaError_t sep_configure(int cfg, int* ctas_per_sm);
bool sep_config_tma_store(int cfg);
// out_tmap: the output tensor map {m, n, batch}, box {128, 2, 1} (TMA-store configs only)
cudaError_t launch_tma_sep(int cfg, bool exact, const CUtensorMap& tmap, const CUtensorMap* out_tmap,
                           const TileGeom& tg, int64_t grid, const float* wv, const float* wh, cudaStream_t stream);
cudaError_t launch_generic_sep(bool exact, const float* in, int64_t in_pitch, int64_t in_image_stride, float* out,
                               int64_t out_pitch, int64_t out_image_stride, int64_t n, int64_t m, int64_t batch,
                               const float* wv, const float* wh, int num_sms, cudaStream_t stream);

// planner / store-mode helpers of harris_abi.cu for other translation units
void plan_tiles_ext(int64_t n, int64_t m, int64_t batch, int64_t gw, int rows_per_stage, int64_t force_rows,
                    TileGeom& tg, int halo);
int store_mode_ext(const float* out, int64_t out_pitch, int64_t batch, int64_t out_image_stride);

// FAST kernel groupings on the strip engine (harris_groupings_tma.cu): the fair fusion ablation
struct GroupLaunchEnv {
    PFN_cuTensorMapEncodeTiled_v12000 encode;
    int num_sms, occ, l2_policy;
};
int64_t grouping_fast_scratch_floats(int grouping, int64_t n, int64_t m);
cudaError_t grouping_fast_configure(int* occ);
int launch_grouping_fast(const GroupLaunchEnv& env, int grouping, float* out, int64_t n, int64_t m, const float* rgb,
                         float* scratch, float kappa, cudaStream_t st);

int64_t grouping_scratch_floats(int grouping, int64_t n, int64_t m);
int grouping_launches(int grouping);
cudaError_t launch_grouping(int grouping, float* out, int64_t n, int64_t m, const float* rgb, float* scratch,
                            float kappa, int num_sms, cudaStream_t stream);

cudaError_t launch_synth(float* dst, int64_t planes, int64_t rows, int64_t W, int64_t dst_pitch,
                         int64_t dst_plane_stride, int64_t H_global, int64_t row0, int64_t plane0,
                         uint64_t seed, int dist, int num_sms, cudaStream_t stream);

// fused-gather completion signalling (harris_peer.cu)
cudaError_t launch_peer_signal(uint32_t* flag, uint32_t epoch, cudaStream_t stream);
cudaError_t launch_peer_wait(const uint32_t* flags, int32_t count, uint32_t epoch, uint32_t* status,
                             int64_t timeout_ns, cudaStream_t stream);

}  // namespace harris
