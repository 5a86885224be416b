// harris_abi.cu — the C-ABI (include/harris_b200.h): device binding, argument
// validation, the tile planner, TMA descriptor encoding, kernel dispatch and the
// pipelined host-buffer path.  Nothing here throws; every entry point returns a
// HARRIS_* code.
//
// Reference boundary being replaced: the thesis host-code convention
// <name>_init / <name>_run / <name>_destroy over the LRA runtime
// and the generated kernel
// harris(output, n0, n1, x0, t1, t2, t3).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost a pointer check unless a tool attaches

#include "../../include/harris_b200.h"
#include "harris_common.cuh"
#include "harris_internal.h"

using namespace harris;

struct harris_ctx {
    int device = 0;
    int num_sms = 0;
    int cc_major = 0, cc_minor = 0;
    int tma_cfg = kDefaultTmaConfig;
    bool tma_cfg_forced = false;  // HARRIS_TMA_CONFIG given: no per-call choice
    int u8_cfg = kDefaultU8Config;
    // register-store config 0: the TMA-store epilogue (config 3) fits only 6 input stages next
    // to its output staging and measured 4 % slower (profiles/sep_store_r02.txt)
    int sep_cfg = 0;
    int occ_sep[kNumSepConfigs] = {0};
    int occ_u8[kNumU8Configs] = {0};
    int occ_ldg[kNumLdgConfigs] = {0};
    int occ_u8ldg = 0;
    int occ_u8bulk = 0;
    int occ_u8pair = 0, occ_u8quad = 0;
    int occ_pair = 0;
    int occ_quad = 0;
    int occ_sepldg = 0;
    int u8ldg_chunk = 0;  // HARRIS_U8LDG_CHUNK: 0 bulk-copy kernel (K1b); 4 / 16-byte cp.async (K2)
    int ldg_cfg = 3;  // HARRIS_LDG_CONFIG; 3 = bulk-copy rows + scalar lane-halo core, 16 warps/SM (K1b:
                      // 404 k MP/s on a column-crop view of 256 x 1080p; the cp.async config 2: 296 k)
    int sync_waves = 1;  // dev knob HARRIS_SYNC_WAVES=0 disables the per-tile CTA barrier
    int sep_bulk = 0;  // HARRIS_SEP_BULK: aligned stencil planes through the bulk-copy kernel too
    // TMA input loads evict_last: the 4-column halo sectors one strip loads are re-read by its
    // neighbour; +0.6-1.3 % over evict_normal on every shape of tools/perf_matrix.sh (f32 batch
    // 413 -> 416 k, 8192^2 398 -> 403 k, u8 886 -> 894 k).  Input lines of a finished launch
    // stay evict_last in L2 until displaced; HARRIS_L2_POLICY=1 restores evict_normal.
    int l2_policy = 2;
    int64_t force_band_rows = 0;  // dev knob (HARRIS_BAND_ROWS): override the planner
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;  // dev knob HARRIS_L2_PROMO
    int occ[kNumTmaConfigs] = {0};
    int occ_win[2] = {0, 0};  // binomial-window kernels of TMA configs 0 and 6
    int occ_grp = 0;          // strip-engine kernel groupings (fusion ablation)
    int pdl_default = 1;      // harris_options.pdl
    int stream_share = 4;     // frames of an independent PDL stream are planned for 1/stream_share of the GPU
                              // (profiles/stream_share_r02.txt: 2-8 within a few %, 16 starves eager launches)
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    std::atomic<int> last_path{HARRIS_PATH_NONE};  // diagnostic; calls may race on different streams
    char last_err[256] = {0};
    // host-buffer pipeline (harris_run_host)
    static constexpr int kSlots = 3;
    cudaStream_t streams[kSlots] = {nullptr, nullptr, nullptr};
    float* d_in[kSlots] = {nullptr, nullptr, nullptr};
    float* d_out[kSlots] = {nullptr, nullptr, nullptr};
    size_t cap_in = 0, cap_out = 0;
    // finished-CTA counter of harris_run_notify (allocated on first use, zeroed; the
    // kernel's last CTA resets it)
    uint32_t* d_notify_counter = nullptr;
    // launch cache: the tensor map, tile plan and grid of the last few distinct call
    // geometries, so a repeated call (a stream of frames, a bench loop) skips the
    // descriptor encode and the planner (~3 us of host time per call)
    struct LaunchEntry {
        bool valid = false;
        int fmt = 0;
        int64_t n = 0, m = 0, batch = 0, in_pitch = 0, in_chan_stride = 0, in_image_stride = 0;
        int64_t out_pitch = 0, out_image_stride = 0;
        const void* rgb = nullptr;
        const void* out = nullptr;
        float kappa = 0.f;
        uint32_t flags = 0;
        int cfg = 0;
        int64_t grid = 0;
        harris::TileGeom tg;
        CUtensorMap tmap;
    };
    static constexpr int kCacheSize = 32;  // a frame ring (harris_run_frames) of up to 32 buffers
    std::mutex cache_mu;
    LaunchEntry cache[kCacheSize];
    int cache_next = 0;
};

namespace {

// NVTX range per C-ABI call (SURVEY.md §5 tracing): library work shows up by name in nsys /
// ncu timelines without the caller instrumenting anything
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Makes ctx->device current for the duration of a call, restores the caller's.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int cuda_fail(harris_ctx* ctx, cudaError_t e, const char* where) {
    if (ctx) std::snprintf(ctx->last_err, sizeof(ctx->last_err), "%s: %s", where, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? HARRIS_ERR_OUT_OF_MEMORY : HARRIS_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// TileGeom::vec_store: 2 = every output row 16-byte aligned (float4 stores); 1 = every row
// 8-byte aligned (two float2 stores per lane: e.g. 1914-float rows); 0 = scalar stores
int32_t store_mode(const float* out, int64_t out_pitch, int64_t batch, int64_t out_image_stride) {
    if (aligned16(out) && (out_pitch & 3) == 0 && (batch == 1 || (out_image_stride & 3) == 0)) return 2;
    if ((reinterpret_cast<uintptr_t>(out) & 7u) == 0 && (out_pitch & 1) == 0 && (batch == 1 || (out_image_stride & 1) == 0))
        return 1;
    return 0;
}

enum Format { kF32Planar = 0, kU8Interleaved = 1 };

struct Call {
    Geom g;
    uint32_t flags;
    int fmt = kF32Planar;  // u8: g.rgb is the byte base, in_pitch / in_image_stride are bytes
    uint32_t* notify_flag = nullptr;  // harris_run_notify
    uint32_t notify_epoch = 0;
    int cfg = -1;  // f32 TMA configuration chosen for this call (resolve_cfg)
    bool ldg = false;  // plan for the cp.async (LDG) kernel
    bool pair = false;  // plan for a row-group TMA kernel (pair- or quad-rows)
    int group = 0;      // rows per group: 2 (pitch = 2 mod 4) or 4 (odd pitch)
};

int validate(const Call& c) {
    const Geom& g = c.g;
    if (!g.rgb || !g.out) return HARRIS_ERR_INVALID_ARGUMENT;
    if (g.n < 1 || g.m < 1) return HARRIS_ERR_SIZE;  // input must be at least 5 x 5
    if (g.n + 4 > INT32_MAX || g.m + 4 > INT32_MAX) return HARRIS_ERR_SIZE;
    if (g.batch < 1) return HARRIS_ERR_INVALID_ARGUMENT;
    if (g.out_pitch < g.m) return HARRIS_ERR_INVALID_ARGUMENT;
    if (g.batch > 1 && g.out_image_stride < g.n * g.out_pitch) return HARRIS_ERR_INVALID_ARGUMENT;
    if (c.fmt == kU8Interleaved) {
        if (g.in_pitch < 3 * (g.m + 4)) return HARRIS_ERR_INVALID_ARGUMENT;
        if (g.batch > 1 && g.in_image_stride < (g.n + 4) * g.in_pitch) return HARRIS_ERR_INVALID_ARGUMENT;
        return HARRIS_OK;
    }
    if (g.in_pitch < g.m + 4) return HARRIS_ERR_INVALID_ARGUMENT;
    if (g.in_chan_stride < (g.n + 4) * g.in_pitch) return HARRIS_ERR_INVALID_ARGUMENT;
    if (g.batch > 1) {
        if (g.in_image_stride < 3 * g.in_chan_stride) return HARRIS_ERR_INVALID_ARGUMENT;
        if (g.out_image_stride < g.n * g.out_pitch) return HARRIS_ERR_INVALID_ARGUMENT;
    }
    return HARRIS_OK;
}

// TMA needs a 16-byte aligned base and 16-byte multiple strides on the INPUT only;
// the output side falls back to scalar stores when its rows are not 16-B aligned.
bool tma_eligible(const Call& c) {
    const Geom& g = c.g;
    if (!aligned16(g.rgb)) return false;
    // the strip engine decodes tiles with 32-bit math: strips per band row < 2^31
    // (tiles = bands x strips/groups stays below that too for any image the TMA box covers)
    if (g.batch * ((g.m + 123) / 124) >= (int64_t(1) << 30)) return false;
    if (c.fmt == kU8Interleaved) {  // byte strides, tensor map over 32-bit words
        if ((g.in_pitch & 15) || (g.batch > 1 && (g.in_image_stride & 15))) return false;
        if (g.batch > INT32_MAX) return false;
        return true;
    }
    if ((g.in_pitch | g.in_chan_stride) & 3) return false;
    if (g.batch > 1 && (g.in_image_stride & 3)) return false;
    const int64_t kMaxStrideBytes = (int64_t(1) << 40) - 16;
    if (g.in_chan_stride * 4 > kMaxStrideBytes) return false;
    if (g.batch > 1 && g.in_image_stride * 4 > kMaxStrideBytes) return false;
    if (g.batch > INT32_MAX) return false;
    return true;
}

// Pick the band height that minimises (waves x rows-per-tile) for a persistent
// grid of `gw` warps: tiles = batch x bands x col_segments.
// Pick the band height that minimises (waves x rows-per-tile) for a persistent grid
// of `gw` warps.  A tile is `groups` 128-column strips: with groups == 2 the strips
// of one band row of all images are paired consecutively (strip_pipeline.cuh).
void plan_tiles(int64_t n, int64_t m, int64_t batch, int64_t gw, int rows_per_stage, int64_t force_rows,
                TileGeom& tg, int halo = 4, int groups = 1, int strip_cols = kWarpCols, bool cap_rows = true,
                int row_align = 1, int64_t max_rows = 288) {
    const int64_t colsegs = (m + strip_cols - 1) / strip_cols;
    const int64_t units_per_band = groups == 2 ? (batch * colsegs + 1) / 2 : batch * colsegs;
    tg.n = int32_t(n);
    tg.m = int32_t(m);
    tg.colsegs = int32_t(colsegs);
    tg.batch = int32_t(batch);
    if (force_rows > 0) {
        const int64_t rows = std::min((force_rows + row_align - 1) / row_align * row_align, n);
        tg.band_rows = int32_t(rows);
        tg.bands = int32_t((n + rows - 1) / rows);
        tg.tiles = units_per_band * tg.bands;
        return;
    }
    const int64_t kTileOverheadRows = 6;  // pipeline/tile switch cost in row-equivalents
    // Tiles taller than this lose more than the cost model sees for the memory-bound ops:
    // the per-tile CTA barrier re-aligns neighbouring strips less often (L2 halo reuse) and
    // the last wave is coarser.  Measured on configs[4]: 538-row tiles 5.12-5.21 ms,
    // 269-row 5.05-5.07 ms; binomial 1076-row 3.48 ms, 269-row 2.97 ms; 32768^2: 886-row
    // 2.526 ms, 254-row 2.517 ms.  The issue-bound u8 op prefers long tiles (1076 rows
    // 2.93-2.95 ms vs 3.03 ms capped) and plans without the cap (profiles/band_rows_r01.txt).
    const int64_t kMaxBandRows = cap_rows ? max_rows : INT64_MAX;
    const int64_t max_bands = std::max<int64_t>(1, std::min<int64_t>(n, 1 + n / 8));
    int64_t best_cost = INT64_MAX, best_rows = n, best_bands = 1;
    for (int64_t nb = 1; nb <= max_bands; ++nb) {
        const int64_t rows = ((n + nb - 1) / nb + row_align - 1) / row_align * row_align;
        const int64_t bands = (n + rows - 1) / rows;
        if (bands != nb) continue;  // same split as a smaller nb
        if (rows > kMaxBandRows && nb < max_bands) continue;
        const int64_t tiles = units_per_band * bands;
        const int64_t waves = (tiles + gw - 1) / gw;
        const int64_t rows_in = ((rows + halo + rows_per_stage - 1) / rows_per_stage) * rows_per_stage;
        const int64_t cost = waves * (rows_in + kTileOverheadRows);
        if (cost < best_cost) {
            best_cost = cost;
            best_rows = rows;
            best_bands = bands;
        }
    }
    tg.band_rows = int32_t(best_rows);
    tg.bands = int32_t(best_bands);
    tg.tiles = units_per_band * best_bands;
}

// f32 inputs TMA cannot describe (pitch / strides / base not 16-byte aligned) keep the
// strip engine with cp.async stage fills; only 4-byte alignment of the floats is needed
bool ldg_eligible(const Call& c) {
    const Geom& g = c.g;
    if (c.fmt == kF32Planar && (reinterpret_cast<uintptr_t>(g.rgb) & 3)) return false;  // u8: any byte address
    if (g.batch * ((g.m + 123) / 124) >= (int64_t(1) << 30)) return false;
    return g.n + 4 <= INT32_MAX && g.m + 4 <= INT32_MAX;
}

// planar f32 whose row pitch is 2 (mod 4) floats: pairs of rows are 16-byte multiples, so a
// tensor map over pair-rows serves it (HarrisF32PairRowOp).  Needs 16-byte aligned planes
// and an even image height (the last pair-row of the last plane must not run past it).
// Returns the rows per group (2 or 4) when a row-group tensor map can serve the call, else 0.
// An odd pitch groups 4 rows (4P floats is a 16-byte multiple): HarrisF32QuadRowOp.
int row_group(const Call& c) {
    const Geom& g = c.g;
    if (!aligned16(g.rgb)) return 0;
    if (c.fmt == kU8Interleaved) {  // byte pitch 8 (mod 16): pairs; 4 (mod 8): quads (K*P % 16 == 0)
        const int k = (g.in_pitch & 15) == 8 ? 2 : (g.in_pitch & 7) == 4 ? 4 : 0;
        if (!k || ((g.n + 4) % k) || (g.batch > 1 && (g.in_image_stride & 15))) return 0;
        if (int64_t(k) * g.in_pitch > INT32_MAX || g.batch > INT32_MAX) return 0;
        return g.batch * ((g.m + 123) / 124) < (int64_t(1) << 30) ? k : 0;
    }
    const int k = (g.in_pitch & 3) == 2 ? 2 : (g.in_pitch & 1) ? 4 : 0;
    if (!k || (g.in_chan_stride & 3) || ((g.n + 4) % k)) return 0;
    if (g.batch > 1 && (g.in_image_stride & 3)) return 0;
    if (int64_t(k) * g.in_pitch > INT32_MAX || g.batch > INT32_MAX) return 0;
    return g.batch * ((g.m + 123) / 124) < (int64_t(1) << 30) ? k : 0;
}
bool pair_eligible(const Call& c) { return row_group(c) != 0; }

int choose_path(const Call& c) {
    if (c.flags & HARRIS_FLAG_FORCE_GENERIC) return HARRIS_PATH_GENERIC;
    // binomial window: the planar-f32 TMA kernels (configs 0 / 6) or the generic kernel
    if (c.flags & HARRIS_FLAG_BINOMIAL_WINDOW)
        return c.fmt == kF32Planar && tma_eligible(c) ? HARRIS_PATH_TMA : HARRIS_PATH_GENERIC;
    if (tma_eligible(c)) return HARRIS_PATH_TMA;
    if (const int k = row_group(c)) return k == 2 ? HARRIS_PATH_PAIR : HARRIS_PATH_QUAD;
    return ldg_eligible(c) ? HARRIS_PATH_LDG : HARRIS_PATH_GENERIC;
}

int pdl_mode(const harris_ctx* ctx, uint32_t flags) {
    return (flags & HARRIS_FLAG_PDL_INDEPENDENT) ? 2 : ((flags & HARRIS_FLAG_PDL) || ctx->pdl_default) ? 1 : 0;
}

constexpr int64_t kStreamFrameMaxPixels = int64_t(16) << 20;  // frames up to 16 MP (4256x2832 = 12 MP)
// internal flag bit (never in the public header): plan an independent frame for the whole GPU —
// harris_run_frames uses it for rings too short to keep stream_share frames in flight, where
// the call boundary (frame 0 waits) would leave the GPU under-filled
constexpr uint32_t kFlagFullGpuPlan = 0x80000000u;

void plan_launch(const harris_ctx* ctx, const Call& c, TileGeom& tg, int64_t& grid) {
    const bool u8 = c.fmt == kU8Interleaved;
    const int fcfg = c.cfg >= 0 ? c.cfg : ctx->tma_cfg;
    const TmaConfig& cfg = c.pair  ? (u8 ? (c.group == 4 ? kU8QuadConfig : kU8PairConfig)
                                         : (c.group == 4 ? kQuadConfig : kPairConfig))
                           : c.ldg ? (u8 ? (ctx->u8ldg_chunk ? kU8LdgConfig : kU8BulkConfig) : kLdgConfigs[ctx->ldg_cfg])
                           : u8    ? kU8Configs[ctx->u8_cfg]
                                   : kTmaConfigs[fcfg];
    const int occ = std::max(1, c.pair  ? (u8 ? (c.group == 4 ? ctx->occ_u8quad : ctx->occ_u8pair)
                                                : (c.group == 4 ? ctx->occ_quad : ctx->occ_pair))
                                : c.ldg ? (u8 ? (ctx->u8ldg_chunk ? ctx->occ_u8ldg : ctx->occ_u8bulk) : ctx->occ_ldg[ctx->ldg_cfg])
                                : u8    ? ctx->occ_u8[ctx->u8_cfg]
                                : c.g.window ? ctx->occ_win[fcfg == 6 ? 1 : 0]
                                        : ctx->occ[fcfg]);
    const int64_t resident_ctas = int64_t(ctx->num_sms) * occ;
    // A single frame of a PDL-independent stream (harris_run_frames, HARRIS_FLAG_PDL_INDEPENDENT)
    // shares the GPU with its neighbours: plan it for 1/kStreamShare of the warps, i.e. fewer,
    // taller tiles (less halo re-read and per-tile overhead) while the next frames fill the
    // other SMs.  Isolated launches keep the whole-GPU plan.
    int64_t plan_warps = resident_ctas * cfg.warps;
    if ((c.flags & HARRIS_FLAG_PDL_INDEPENDENT) && !(c.flags & kFlagFullGpuPlan) && c.g.batch == 1 &&
        (c.g.n + 4) * (c.g.m + 4) <= kStreamFrameMaxPixels)
        plan_warps = std::max<int64_t>(cfg.warps, plan_warps / ctx->stream_share);
    // u8 ops sum the box rows in pairs (kPairRows) by the row's parity within the stage: even
    // tile heights keep every tile start on an even absolute row, so the pairing — and the FAST
    // bits — do not depend on the tile plan (f32 ops do not pair rows)
    plan_tiles(c.g.n, c.g.m, c.g.batch, plan_warps, cfg.rows, ctx->force_band_rows, tg, 4,
               cfg.groups, cfg.strip_cols, /*cap_rows=*/!u8, /*row_align=*/c.pair ? c.group : u8 ? 2 : 1);
    grid = std::min<int64_t>((tg.tiles + cfg.warps - 1) / cfg.warps, resident_ctas);
    tg.out = c.g.out;
    tg.out_pitch = c.g.out_pitch;
    tg.out_image_stride = c.g.out_image_stride;
    tg.kappa = c.g.kappa;
    tg.l2_policy = ctx->l2_policy;
    tg.vec_store = store_mode(c.g.out, c.g.out_pitch, c.g.batch, c.g.out_image_stride);
    tg.sync_waves = ctx->sync_waves;
    tg.pdl = pdl_mode(ctx, c.flags);
}

// Short tiles (a small image fills the GPU with a few rows per warp): the pipeline ramp
// dominates and the scalar single-strip core over all SMs beats the packed dual-strip
// core (configs[1] 1536x2560: 18.5 vs 20.5 us, profiles/small_image_probe_r01.txt).
constexpr int kShortTileRows = 32;
constexpr int kShortTileTmaConfig = 0;

int resolve_cfg(const harris_ctx* ctx, const Call& c) {
    if (c.fmt == kU8Interleaved || ctx->tma_cfg_forced) return ctx->tma_cfg;
    Call probe = c;
    probe.cfg = ctx->tma_cfg;
    TileGeom tg;
    int64_t grid = 0;
    plan_launch(ctx, probe, tg, grid);
    return tg.band_rows < kShortTileRows ? kShortTileTmaConfig : ctx->tma_cfg;
}

int encode_tmap_u8(harris_ctx* ctx, const Call& c, CUtensorMap* tmap) {
    const Geom& g = c.g;
    const TmaConfig& cfg = kU8Configs[ctx->u8_cfg];
    cuuint64_t dims[3] = {cuuint64_t((3 * (g.m + 4) + 3) / 4), cuuint64_t(g.n + 4), cuuint64_t(g.batch)};
    const int64_t img_stride = g.batch > 1 ? g.in_image_stride : (g.n + 4) * g.in_pitch;
    cuuint64_t strides[2] = {cuuint64_t(g.in_pitch), cuuint64_t((img_stride + 15) / 16 * 16)};
    cuuint32_t box[3] = {cuuint32_t(kU8BoxWords), cuuint32_t(cfg.rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = ctx->encode(tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<float*>(g.rgb), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             ctx->promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled (u8) failed (CUresult %d)",
                      int(r));
        return HARRIS_ERR_TMA;
    }
    return HARRIS_OK;
}

// row-group view of planar f32 (K = 2 for pitch P = 2 mod 4, K = 4 for odd P):
// {K*P columns, H/K groups, 3, B}
int encode_tmap_pair(harris_ctx* ctx, const Call& c, CUtensorMap* tmap) {
    const Geom& g = c.g;
    const int64_t k = c.group;
    cuuint64_t dims[4] = {cuuint64_t(k * g.in_pitch), cuuint64_t((g.n + 4) / k), 3, cuuint64_t(g.batch)};
    const int64_t img_stride = g.batch > 1 ? g.in_image_stride : 3 * g.in_chan_stride;
    cuuint64_t strides[3] = {cuuint64_t(k * g.in_pitch) * 4, cuuint64_t(g.in_chan_stride) * 4,
                             cuuint64_t(img_stride) * 4};
    cuuint32_t box[4] = {132, 3, 3, 1};  // HarrisF32PairRowOp::kRow
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = ctx->encode(tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(g.rgb), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, ctx->promo,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled (pair) failed (CUresult %d)",
                      int(r));
        return HARRIS_ERR_TMA;
    }
    return HARRIS_OK;
}

// row-group view of interleaved u8 (K = 2 / 4 rows): {K*P/4 words, H/K groups, B}
int encode_tmap_u8_group(harris_ctx* ctx, const Call& c, CUtensorMap* tmap) {
    const Geom& g = c.g;
    const int64_t k = c.group;
    cuuint64_t dims[3] = {cuuint64_t(k * g.in_pitch / 4), cuuint64_t((g.n + 4) / k), cuuint64_t(g.batch)};
    const int64_t img_stride = g.batch > 1 ? g.in_image_stride : (g.n + 4) * g.in_pitch;
    cuuint64_t strides[2] = {cuuint64_t(k * g.in_pitch), cuuint64_t(img_stride)};
    cuuint32_t box[3] = {cuuint32_t(kU8BoxWords), cuuint32_t((k == 2 ? 6 : 12) / k), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = ctx->encode(tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<float*>(g.rgb), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, ctx->promo,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled (u8 rows) failed (CUresult %d)",
                      int(r));
        return HARRIS_ERR_TMA;
    }
    return HARRIS_OK;
}

int encode_tmap(harris_ctx* ctx, const Call& c, CUtensorMap* tmap) {
    if (c.fmt == kU8Interleaved) return c.pair ? encode_tmap_u8_group(ctx, c, tmap) : encode_tmap_u8(ctx, c, tmap);
    if (c.pair) return encode_tmap_pair(ctx, c, tmap);
    const Geom& g = c.g;
    const TmaConfig& cfg = kTmaConfigs[c.cfg >= 0 ? c.cfg : ctx->tma_cfg];
    cuuint64_t dims[4] = {cuuint64_t(g.m + 4), cuuint64_t(g.n + 4), 3, cuuint64_t(g.batch)};
    const int64_t img_stride = g.batch > 1 ? g.in_image_stride : 3 * g.in_chan_stride;
    cuuint64_t strides[3] = {cuuint64_t(g.in_pitch) * 4, cuuint64_t(g.in_chan_stride) * 4,
                             cuuint64_t(img_stride) * 4};
    cuuint32_t box[4] = {cuuint32_t(cfg.strip_cols + 4), cuuint32_t(cfg.rows), 3, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = ctx->encode(tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(g.rgb), dims, strides,
                             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             ctx->promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled failed (CUresult %d)", int(r));
        return HARRIS_ERR_TMA;
    }
    return HARRIS_OK;
}

bool cache_match(const harris_ctx::LaunchEntry& e, const Call& c) {
    const Geom& g = c.g;
    return e.valid && e.fmt == c.fmt && e.n == g.n && e.m == g.m && e.batch == g.batch && e.rgb == g.rgb &&
           e.in_pitch == g.in_pitch && e.in_chan_stride == g.in_chan_stride &&
           e.in_image_stride == g.in_image_stride && e.out == g.out && e.out_pitch == g.out_pitch &&
           e.out_image_stride == g.out_image_stride && e.kappa == g.kappa && e.flags == c.flags;
}

bool cache_lookup(harris_ctx* ctx, const Call& c, harris_ctx::LaunchEntry& out) {
    std::lock_guard<std::mutex> lock(ctx->cache_mu);
    for (const auto& e : ctx->cache) {
        if (cache_match(e, c)) {
            out = e;
            return true;
        }
    }
    return false;
}

void cache_insert(harris_ctx* ctx, const Call& c, harris_ctx::LaunchEntry ent) {
    const Geom& g = c.g;
    ent.valid = true;
    ent.fmt = c.fmt;
    ent.n = g.n;
    ent.m = g.m;
    ent.batch = g.batch;
    ent.rgb = g.rgb;
    ent.in_pitch = g.in_pitch;
    ent.in_chan_stride = g.in_chan_stride;
    ent.in_image_stride = g.in_image_stride;
    ent.out = g.out;
    ent.out_pitch = g.out_pitch;
    ent.out_image_stride = g.out_image_stride;
    ent.kappa = g.kappa;
    ent.flags = c.flags;
    std::lock_guard<std::mutex> lock(ctx->cache_mu);
    ctx->cache[ctx->cache_next] = ent;
    ctx->cache_next = (ctx->cache_next + 1) % harris_ctx::kCacheSize;
}

int run(harris_ctx* ctx, const Call& c, cudaStream_t stream) {
    if (!ctx) return HARRIS_ERR_INVALID_ARGUMENT;
    NvtxRange nvtx(c.fmt == kU8Interleaved ? "harris_run_u8" : "harris_run");
    int rc = validate(c);
    if (rc) return rc;
    const bool exact = (c.flags & HARRIS_FLAG_EXACT_ORDER) != 0;
    int path = choose_path(c);
    if (path != HARRIS_PATH_TMA && (c.flags & HARRIS_FLAG_FORCE_TMA)) return HARRIS_ERR_ALIGNMENT;
    DeviceGuard guard(ctx->device);
    if (!guard.ok) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
    cudaError_t e;
    if (path == HARRIS_PATH_TMA || path == HARRIS_PATH_LDG || path == HARRIS_PATH_PAIR ||
        path == HARRIS_PATH_QUAD) {
        const bool ldg = path == HARRIS_PATH_LDG;
        const bool pair = path == HARRIS_PATH_PAIR || path == HARRIS_PATH_QUAD;
        const int group = path == HARRIS_PATH_QUAD ? 4 : 2;
        harris_ctx::LaunchEntry ent;
        if (!cache_lookup(ctx, c, ent)) {
            Call cc = c;
            cc.ldg = ldg;
            cc.pair = pair;
            cc.group = group;
            if (!ldg) {
                cc.cfg = pair ? 0 : resolve_cfg(ctx, c);
                if (c.g.window && !tma_window_config(cc.cfg)) cc.cfg = kTmaConfigs[cc.cfg].groups == 2 ? 6 : 0;
                rc = encode_tmap(ctx, cc, &ent.tmap);
                if (rc) return rc;
            }
            plan_launch(ctx, cc, ent.tg, ent.grid);
            ent.cfg = cc.cfg;
            if (ent.tg.tiles > INT32_MAX) return HARRIS_ERR_SIZE;  // beyond the engine's 32-bit tile index
            cache_insert(ctx, c, ent);
        }
        TileGeom tg = ent.tg;
        if (c.notify_flag) {
            tg.notify_counter = ctx->d_notify_counter;
            tg.notify_flag = c.notify_flag;
            tg.notify_epoch = c.notify_epoch;
        }
        e = pair ? (c.fmt == kU8Interleaved
                        ? launch_tma_u8_group(group, exact, ent.tmap, tg, ent.grid, int32_t(c.g.in_pitch / 4), stream)
                    : group == 4 ? launch_tma_quad(exact, ent.tmap, tg, ent.grid, int32_t(c.g.in_pitch), stream)
                                 : launch_tma_pair(exact, ent.tmap, tg, ent.grid, int32_t(c.g.in_pitch), stream))
            : ldg ? (c.fmt == kU8Interleaved ? launch_u8_ldg(exact, ctx->u8ldg_chunk, c.g, tg, ent.grid, stream)
                                             : launch_ldg(ctx->ldg_cfg, exact, c.g, tg, ent.grid, stream))
            : c.fmt == kU8Interleaved ? launch_tma_u8(ctx->u8_cfg, exact, ent.tmap, tg, ent.grid, stream)
            : c.g.window              ? launch_tma_window(ent.cfg, exact, ent.tmap, tg, ent.grid, stream)
                                      : launch_tma(ent.cfg, exact, ent.tmap, tg, ent.grid, stream);
    } else {
        e = c.fmt == kU8Interleaved ? launch_generic_u8(exact, c.g, stream) : launch_generic(exact, c.g, stream);
        if (e == cudaSuccess && c.notify_flag) e = launch_peer_signal(c.notify_flag, c.notify_epoch, stream);
    }
    if (e != cudaSuccess)
        return cuda_fail(ctx, e, path == HARRIS_PATH_TMA    ? "launch tma"
                                 : path == HARRIS_PATH_PAIR ? "launch tma pair"
                                 : path == HARRIS_PATH_QUAD ? "launch tma quad"
                                 : path == HARRIS_PATH_LDG  ? "launch ldg"
                                                            : "launch generic");
    ctx->last_path = path;
    return HARRIS_OK;
}

Call make_call(float* out, int64_t out_pitch, int64_t out_image_stride, int64_t n, int64_t m, const float* rgb,
               int64_t in_pitch, int64_t in_chan_stride, int64_t in_image_stride, int64_t batch, float kappa,
               uint32_t flags) {
    Call c;
    c.g.n = n;
    c.g.m = m;
    c.g.batch = batch;
    c.g.rgb = rgb;
    c.g.in_pitch = in_pitch;
    c.g.in_chan_stride = in_chan_stride;
    c.g.in_image_stride = in_image_stride;
    c.g.out = out;
    c.g.out_pitch = out_pitch;
    c.g.out_image_stride = out_image_stride;
    c.g.kappa = kappa;
    c.g.window = (flags & HARRIS_FLAG_BINOMIAL_WINDOW) ? 1 : 0;
    c.flags = flags;
    return c;
}

}  // namespace

namespace harris {
void plan_tiles_ext(int64_t n, int64_t m, int64_t batch, int64_t gw, int rows_per_stage, int64_t force_rows,
                    TileGeom& tg, int halo) {
    plan_tiles(n, m, batch, gw, rows_per_stage, force_rows, tg, halo);
}

int store_mode_ext(const float* out, int64_t out_pitch, int64_t batch, int64_t out_image_stride) {
    return store_mode(out, out_pitch, batch, out_image_stride);
}
}  // namespace harris

extern "C" {

int harris_abi_version(void) { return HARRIS_B200_ABI_VERSION; }

const char* harris_strerror(int code) {
    switch (code) {
        case HARRIS_OK: return "ok";
        case HARRIS_ERR_INVALID_ARGUMENT: return "invalid argument (null pointer, pitch, stride or batch)";
        case HARRIS_ERR_SIZE: return "invalid size (input must be at least 5x5: n >= 1, m >= 1)";
        case HARRIS_ERR_ALIGNMENT: return "TMA path requested but data is not 16-byte aligned";
        case HARRIS_ERR_CUDA: return "CUDA runtime error";
        case HARRIS_ERR_NO_DEVICE: return "no CUDA device";
        case HARRIS_ERR_TMA: return "TMA descriptor encoding failed";
        case HARRIS_ERR_OUT_OF_MEMORY: return "out of device memory";
        case HARRIS_ERR_UNSUPPORTED_DEVICE: return "unsupported device (needs sm_100 / B200)";
        default: return "unknown error";
    }
}

void harris_options_default(harris_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->struct_size = uint32_t(sizeof(harris_options));
    o->l2_policy = HARRIS_L2_EVICT_LAST;
    o->band_rows = 0;
    o->pdl = 1;
}

int harris_init(harris_ctx** out_ctx, int cuda_device) { return harris_init_ex(out_ctx, cuda_device, nullptr); }

int harris_init_ex(harris_ctx** out_ctx, int cuda_device, const harris_options* opts) {
    if (!out_ctx) return HARRIS_ERR_INVALID_ARGUMENT;
    *out_ctx = nullptr;
    harris_options o;
    harris_options_default(&o);
    if (opts) {
        if (opts->struct_size < uint32_t(offsetof(harris_options, reserved))) return HARRIS_ERR_INVALID_ARGUMENT;
        if (opts->l2_policy < HARRIS_L2_EVICT_FIRST || opts->l2_policy > HARRIS_L2_EVICT_LAST) return HARRIS_ERR_INVALID_ARGUMENT;
        if (opts->band_rows < 0 || opts->pdl < 0 || opts->pdl > 1) return HARRIS_ERR_INVALID_ARGUMENT;
        o.l2_policy = opts->l2_policy;
        o.band_rows = opts->band_rows;
        o.pdl = opts->pdl;
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return HARRIS_ERR_NO_DEVICE;
    }
    int dev = cuda_device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return HARRIS_ERR_NO_DEVICE;
    if (dev >= count) return HARRIS_ERR_NO_DEVICE;
    harris_ctx* ctx = new (std::nothrow) harris_ctx();
    if (!ctx) return HARRIS_ERR_OUT_OF_MEMORY;
    ctx->device = dev;
    DeviceGuard guard(dev);
    cudaDeviceProp prop;
    if (!guard.ok || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
        delete ctx;
        return HARRIS_ERR_NO_DEVICE;
    }
    ctx->num_sms = prop.multiProcessorCount;
    ctx->cc_major = prop.major;
    ctx->cc_minor = prop.minor;
    if (prop.major != 10) {  // binary carries sm_100a SASS only
        delete ctx;
        return HARRIS_ERR_UNSUPPORTED_DEVICE;
    }
    ctx->l2_policy = o.l2_policy;
    ctx->force_band_rows = o.band_rows;
    ctx->pdl_default = o.pdl;
    // Developer knobs (kernel configuration, tiling, L2 promotion / policy): read only with
    // HARRIS_DEV=1 so a drop-in library never changes behaviour from the environment.
    const char* dev_env = std::getenv("HARRIS_DEV");
    if (dev_env && std::atoi(dev_env) == 1) {
        const char* env = std::getenv("HARRIS_TMA_CONFIG");
        if (env) {
            int v = std::atoi(env);
            if (v >= 0 && v < kNumTmaConfigs) {
                ctx->tma_cfg = v;
                ctx->tma_cfg_forced = true;
            }
        }
        env = std::getenv("HARRIS_U8_CONFIG");
        if (env) {
            int v = std::atoi(env);
            if (v >= 0 && v < kNumU8Configs) ctx->u8_cfg = v;
        }
        env = std::getenv("HARRIS_SEP_BULK");
        if (env) ctx->sep_bulk = std::atoi(env) != 0;
        env = std::getenv("HARRIS_SEP_CONFIG");
        if (env) {
            int v = std::atoi(env);
            if (v >= 0 && v < kNumSepConfigs) ctx->sep_cfg = v;
        }
        env = std::getenv("HARRIS_U8LDG_CHUNK");
        if (env) ctx->u8ldg_chunk = std::atoi(env) == 4 ? 4 : std::atoi(env) == 16 ? 16 : 0;
        env = std::getenv("HARRIS_LDG_CONFIG");
        if (env) {
            int v = std::atoi(env);
            if (v >= 0 && v < kNumLdgConfigs) ctx->ldg_cfg = v;
        }
        env = std::getenv("HARRIS_SYNC_WAVES");
        if (env) ctx->sync_waves = std::atoi(env) != 0;
        env = std::getenv("HARRIS_L2_PROMO");
        if (env) {
            const int v = std::atoi(env);
            const CUtensorMapL2promotion tab[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
            if (v >= 0 && v < 4) ctx->promo = tab[v];
        }
        env = std::getenv("HARRIS_BAND_ROWS");
        if (env) ctx->force_band_rows = std::atoll(env);
        env = std::getenv("HARRIS_STREAM_SHARE");
        if (env && std::atoi(env) >= 1) ctx->stream_share = std::atoi(env);
        env = std::getenv("HARRIS_L2_POLICY");
        if (env) {
            int v = std::atoi(env);
            if (v >= 0 && v <= 2) ctx->l2_policy = v;
        }
    }
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
        int rc = cuda_fail(ctx, e, "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        delete ctx;
        return rc;
    }
    ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    for (int k = 0; k < kNumTmaConfigs; ++k) {
        e = tma_configure(k);
        if (e == cudaSuccess) e = tma_occupancy(k, &ctx->occ[k]);
        if (e != cudaSuccess) {
            int rc = cuda_fail(ctx, e, "configure tma kernel");
            delete ctx;
            return rc;
        }
    }
    if (e == cudaSuccess) e = tma_window_configure();
    if (e == cudaSuccess) e = tma_window_occupancy(0, &ctx->occ_win[0]);
    if (e == cudaSuccess) e = tma_window_occupancy(6, &ctx->occ_win[1]);
    if (e == cudaSuccess) e = grouping_fast_configure(&ctx->occ_grp);
    e = e == cudaSuccess ? pair_configure(&ctx->occ_pair) : e;
    if (e == cudaSuccess) e = quad_configure(&ctx->occ_quad);
    if (e == cudaSuccess) e = sep_ldg_configure(&ctx->occ_sepldg);
    if (e == cudaSuccess) e = u8_ldg_configure(&ctx->occ_u8ldg, &ctx->occ_u8bulk);
    if (e == cudaSuccess) e = u8_group_configure(&ctx->occ_u8pair, &ctx->occ_u8quad);
    if (e != cudaSuccess) {
        int rc = cuda_fail(ctx, e, "configure u8 ldg kernel");
        delete ctx;
        return rc;
    }
    for (int k = 0; k < kNumLdgConfigs; ++k) {
        e = ldg_configure(k, &ctx->occ_ldg[k]);
        if (e != cudaSuccess) {
            int rc = cuda_fail(ctx, e, "configure ldg kernel");
            delete ctx;
            return rc;
        }
    }
    for (int k = 0; k < kNumSepConfigs; ++k) {
        e = sep_configure(k, &ctx->occ_sep[k]);
        if (e != cudaSuccess) {
            int rc = cuda_fail(ctx, e, "configure stencil kernel");
            delete ctx;
            return rc;
        }
    }
    for (int k = 0; k < kNumU8Configs; ++k) {
        e = u8_configure(k);
        if (e == cudaSuccess) e = u8_occupancy(k, &ctx->occ_u8[k]);
        if (e != cudaSuccess) {
            int rc = cuda_fail(ctx, e, "configure u8 tma kernel");
            delete ctx;
            return rc;
        }
    }
    *out_ctx = ctx;
    return HARRIS_OK;
}

void harris_destroy(harris_ctx* ctx) {
    if (!ctx) return;
    {
        DeviceGuard guard(ctx->device);
        for (int k = 0; k < harris_ctx::kSlots; ++k) {
            if (ctx->streams[k]) {
                cudaStreamSynchronize(ctx->streams[k]);
                cudaStreamDestroy(ctx->streams[k]);
            }
            cudaFree(ctx->d_in[k]);
            cudaFree(ctx->d_out[k]);
        }
        cudaFree(ctx->d_notify_counter);
    }
    delete ctx;
}

int harris_run(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t n, int64_t m, const float* rgb, float kappa,
               void* stream) {
    const int64_t W = m + 4, H = n + 4;
    return run(ctx, make_call(out, out_pitch, n * out_pitch, n, m, rgb, W, H * W, 3 * H * W, 1, kappa, 0),
               static_cast<cudaStream_t>(stream));
}

int harris_run_batched(harris_ctx* ctx, float* out, int64_t n, int64_t m, const float* rgb, int64_t batch,
                       float kappa, void* stream) {
    const int64_t W = m + 4, H = n + 4;
    return run(ctx, make_call(out, m, n * m, n, m, rgb, W, H * W, 3 * H * W, batch, kappa, 0),
               static_cast<cudaStream_t>(stream));
}

int harris_run_strided(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride, int64_t n,
                       int64_t m, const float* rgb, int64_t in_pitch, int64_t in_chan_stride,
                       int64_t in_image_stride, int64_t batch, float kappa, uint32_t flags, void* stream) {
    return run(ctx,
               make_call(out, out_pitch, out_image_stride, n, m, rgb, in_pitch, in_chan_stride, in_image_stride,
                         batch, kappa, flags),
               static_cast<cudaStream_t>(stream));
}

// shared body of harris_run_frames / harris_run_frames_u8
static int run_frames_impl(harris_ctx* ctx, int fmt, float* const* outs, int64_t out_pitch, int64_t n, int64_t m,
                           const void* const* ins, int64_t in_pitch, int64_t in_chan_stride, int64_t frames,
                           float kappa, uint32_t flags, void* stream) {
    if (!ctx || !outs || !ins || frames < 1) return HARRIS_ERR_INVALID_ARGUMENT;
    // frames 1.. run as independent of their predecessors: their outputs must be distinct
    // (checked for rings of up to 256 frames; larger rings are the caller's contract)
    if (frames <= 256)
        for (int64_t a = 0; a < frames; ++a)
            for (int64_t b = a + 1; b < frames; ++b)
                if (outs[a] == outs[b]) return HARRIS_ERR_INVALID_ARGUMENT;
    uint32_t base = flags & ~(uint32_t(HARRIS_FLAG_PDL) | uint32_t(HARRIS_FLAG_PDL_INDEPENDENT) | kFlagFullGpuPlan);
    if (frames < 2 * int64_t(ctx->stream_share)) base |= kFlagFullGpuPlan;
    NvtxRange nvtx(fmt == kU8Interleaved ? "harris_run_frames_u8" : "harris_run_frames");
    for (int64_t k = 0; k < frames; ++k) {
        const uint32_t pdl = k > 0 || (flags & HARRIS_FLAG_PDL_INDEPENDENT) ? HARRIS_FLAG_PDL_INDEPENDENT
                                                                            : HARRIS_FLAG_PDL;
        if (!ins[k]) return HARRIS_ERR_INVALID_ARGUMENT;
        Call c = fmt == kU8Interleaved
                     ? make_call(outs[k], out_pitch, n * out_pitch, n, m, static_cast<const float*>(ins[k]), in_pitch,
                                 0, (n + 4) * in_pitch, 1, kappa, base | pdl)
                     : make_call(outs[k], out_pitch, n * out_pitch, n, m, static_cast<const float*>(ins[k]), in_pitch,
                                 in_chan_stride, 3 * in_chan_stride, 1, kappa, base | pdl);
        c.fmt = fmt;
        const int rc = run(ctx, c, static_cast<cudaStream_t>(stream));
        if (rc) return rc;
    }
    return HARRIS_OK;
}

int harris_run_frames(harris_ctx* ctx, float* const* outs, int64_t out_pitch, int64_t n, int64_t m,
                      const float* const* rgbs, int64_t in_pitch, int64_t in_chan_stride, int64_t frames,
                      float kappa, uint32_t flags, void* stream) {
    return run_frames_impl(ctx, kF32Planar, outs, out_pitch, n, m, reinterpret_cast<const void* const*>(rgbs),
                           in_pitch, in_chan_stride, frames, kappa, flags, stream);
}

int harris_run_frames_u8(harris_ctx* ctx, float* const* outs, int64_t out_pitch, int64_t n, int64_t m,
                         const uint8_t* const* rgb8s, int64_t in_pitch_bytes, int64_t frames, float kappa,
                         uint32_t flags, void* stream) {
    return run_frames_impl(ctx, kU8Interleaved, outs, out_pitch, n, m, reinterpret_cast<const void* const*>(rgb8s),
                           in_pitch_bytes, 0, frames, kappa, flags, stream);
}

int harris_run_notify(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride, int64_t n,
                      int64_t m, const float* rgb, int64_t in_pitch, int64_t in_chan_stride, int64_t in_image_stride,
                      int64_t batch, float kappa, uint32_t flags, uint32_t* notify_flag, uint32_t epoch,
                      void* stream) {
    if (!ctx || !notify_flag) return HARRIS_ERR_INVALID_ARGUMENT;
    if (!ctx->d_notify_counter) {
        DeviceGuard guard(ctx->device);
        if (!guard.ok) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
        cudaError_t e = cudaMalloc(&ctx->d_notify_counter, sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMemset(ctx->d_notify_counter, 0, sizeof(uint32_t));
        if (e != cudaSuccess) {
            cudaFree(ctx->d_notify_counter);
            ctx->d_notify_counter = nullptr;
            return cuda_fail(ctx, e, "notify counter");
        }
    }
    Call c = make_call(out, out_pitch, out_image_stride, n, m, rgb, in_pitch, in_chan_stride, in_image_stride, batch,
                       kappa, flags);
    c.notify_flag = notify_flag;
    c.notify_epoch = epoch;
    return run(ctx, c, static_cast<cudaStream_t>(stream));
}

int harris_run_u8(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride, int64_t n, int64_t m,
                  const uint8_t* rgb8, int64_t in_pitch_bytes, int64_t in_image_stride_bytes, int64_t batch,
                  float kappa, uint32_t flags, void* stream) {
    Call c = make_call(out, out_pitch, out_image_stride, n, m, reinterpret_cast<const float*>(rgb8), in_pitch_bytes,
                       0, in_image_stride_bytes, batch, kappa, flags);
    c.fmt = kU8Interleaved;
    if (!rgb8) return HARRIS_ERR_INVALID_ARGUMENT;
    return run(ctx, c, static_cast<cudaStream_t>(stream));
}

int harris_stencil3x3_sep(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride, int64_t n,
                          int64_t m, const float* in, int64_t in_pitch, int64_t in_image_stride, int64_t batch,
                          const float* wv, const float* wh, uint32_t flags, void* stream_) {
    if (!ctx || !out || !in || !wv || !wh) return HARRIS_ERR_INVALID_ARGUMENT;
    if (n < 1 || m < 1) return HARRIS_ERR_SIZE;
    if (n + 2 > INT32_MAX || m + 2 > INT32_MAX) return HARRIS_ERR_SIZE;
    NvtxRange nvtx("harris_stencil3x3_sep");
    if (batch < 1 || in_pitch < m + 2 || out_pitch < m) return HARRIS_ERR_INVALID_ARGUMENT;
    if (batch > 1 && (in_image_stride < (n + 2) * in_pitch || out_image_stride < n * out_pitch))
        return HARRIS_ERR_INVALID_ARGUMENT;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const bool exact = (flags & HARRIS_FLAG_EXACT_ORDER) != 0;
    const int64_t img_stride = batch > 1 ? in_image_stride : (n + 2) * in_pitch;
    const bool tma_ok = !(flags & HARRIS_FLAG_FORCE_GENERIC) && aligned16(in) && (in_pitch & 3) == 0 &&
                        (batch == 1 || (in_image_stride & 3) == 0) && batch <= INT32_MAX;
    if (!tma_ok && (flags & HARRIS_FLAG_FORCE_TMA)) return HARRIS_ERR_ALIGNMENT;
    // aligned planes too go through the bulk-copy kernel when ctx->sep_bulk (HARRIS_SEP_BULK)
    const bool tma = tma_ok && (!ctx->sep_bulk || (flags & HARRIS_FLAG_FORCE_TMA));
    // other 4-byte aligned planes: the same strip engine with cp.async stage fills
    const bool ldg = !tma && !(flags & HARRIS_FLAG_FORCE_GENERIC) && (reinterpret_cast<uintptr_t>(in) & 3) == 0 &&
                     batch * ((m + 127) / 128) < (int64_t(1) << 30);
    DeviceGuard guard(ctx->device);
    if (!guard.ok) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
    cudaError_t e;
    if (ldg) {
        TileGeom tg;
        const int64_t resident = int64_t(ctx->num_sms) * std::max(1, ctx->occ_sepldg);
        plan_tiles(n, m, batch, resident * kSepLdgConfig.warps, kSepLdgConfig.rows, ctx->force_band_rows, tg, 2);
        const int64_t grid = std::min<int64_t>((tg.tiles + kSepLdgConfig.warps - 1) / kSepLdgConfig.warps, resident);
        tg.out = out;
        tg.out_pitch = out_pitch;
        tg.out_image_stride = batch > 1 ? out_image_stride : n * out_pitch;
        tg.kappa = 0.f;
        tg.l2_policy = ctx->l2_policy;
        tg.vec_store = store_mode(out, out_pitch, batch, out_image_stride);
        tg.sync_waves = ctx->sync_waves;
        tg.pdl = pdl_mode(ctx, flags);
        if (tg.tiles > INT32_MAX) return HARRIS_ERR_SIZE;
        e = launch_sep_ldg(exact, in, in_pitch, img_stride, m + 2, n + 2, tg, grid, wv, wh, stream);
    } else if (tma) {
        CUtensorMap tmap;
        cuuint64_t dims[3] = {cuuint64_t(m + 2), cuuint64_t(n + 2), cuuint64_t(batch)};
        cuuint64_t strides[2] = {cuuint64_t(in_pitch) * 4, cuuint64_t((img_stride + 3) / 4 * 4) * 4};
        const int out_vec = store_mode(out, out_pitch, batch, out_image_stride);
        // TMA-store epilogue: needs 16-byte aligned output rows / images (tensor-map strides) and
        // m % 4 == 0 — a TMA store writes the out-of-bounds tail of a box's last 16-byte chunk
        // (measured: m = 6 wrote columns 6 and 7), which would touch the caller's padding
        const int cfg = sep_config_tma_store(ctx->sep_cfg) && (out_vec != 2 || (m & 3)) ? 0 : ctx->sep_cfg;
        const TmaConfig& scfg = kSepConfigs[cfg];
        cuuint32_t box[3] = {cuuint32_t(kBoxCols), cuuint32_t(scfg.rows), 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = ctx->encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 ctx->promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled (stencil) failed (%d)", int(r));
            return HARRIS_ERR_TMA;
        }
        TileGeom tg;
        const int64_t resident = int64_t(ctx->num_sms) * std::max(1, ctx->occ_sep[cfg]);
        // TMA stores: row pairs never straddle tiles.  Tiles of at most 136 rows: the 8 warps of a
        // CTA re-align at every tile boundary, which this 1:1 read/write op needs more than the
        // Harris ops (1024 x 1080x1920: 269-row tiles 710 k MP/s, 136-row 796 k; 16 x 8192^2
        // 680 -> 695 k; 256 x 1536x2560 771 -> 788 k; profiles/band_rows_r02.txt)
        plan_tiles(n, m, batch, resident * scfg.warps, scfg.rows, ctx->force_band_rows, tg, 2, 1, kWarpCols, true,
                   sep_config_tma_store(cfg) ? 2 : 1, kSepMaxBandRows);
        const int64_t grid = std::min<int64_t>((tg.tiles + scfg.warps - 1) / scfg.warps, resident);
        tg.out = out;
        tg.out_pitch = out_pitch;
        tg.out_image_stride = batch > 1 ? out_image_stride : n * out_pitch;
        tg.kappa = 0.f;
        tg.l2_policy = ctx->l2_policy;
        tg.vec_store = out_vec;
        tg.sync_waves = ctx->sync_waves;
        tg.pdl = pdl_mode(ctx, flags);
        if (tg.tiles > INT32_MAX) return HARRIS_ERR_SIZE;  // beyond the engine's 32-bit tile index
        CUtensorMap out_tmap;
        const bool ts = sep_config_tma_store(cfg);
        if (ts) {
            cuuint64_t odims[3] = {cuuint64_t(m), cuuint64_t(n), cuuint64_t(batch)};
            cuuint64_t ostr[2] = {cuuint64_t(out_pitch) * 4, cuuint64_t(batch > 1 ? out_image_stride : n * out_pitch) * 4};
            cuuint32_t obox[3] = {cuuint32_t(kWarpCols), 2, 1};
            r = ctx->encode(&out_tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, odims, ostr, obox, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled (stencil out) failed (%d)",
                              int(r));
                return HARRIS_ERR_TMA;
            }
        }
        e = launch_tma_sep(cfg, exact, tmap, ts ? &out_tmap : nullptr, tg, grid, wv, wh, stream);
    } else {
        e = launch_generic_sep(exact, in, in_pitch, img_stride, out, out_pitch,
                               batch > 1 ? out_image_stride : n * out_pitch, n, m, batch, wv, wh, ctx->num_sms,
                               stream);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch stencil");
    ctx->last_path = tma ? HARRIS_PATH_TMA : ldg ? HARRIS_PATH_LDG : HARRIS_PATH_GENERIC;
    return HARRIS_OK;
}

int harris_plan(harris_ctx* ctx, int64_t n, int64_t m, int64_t batch, const float* rgb, int64_t in_pitch,
                int64_t in_chan_stride, int64_t in_image_stride, const float* out, int64_t out_pitch,
                int64_t out_image_stride, uint32_t flags, harris_plan_info* info) {
    if (!ctx || !info) return HARRIS_ERR_INVALID_ARGUMENT;
    Call c = make_call(const_cast<float*>(out), out_pitch, out_image_stride, n, m, rgb, in_pitch, in_chan_stride,
                       in_image_stride, batch, 0.04f, flags);
    int rc = validate(c);
    if (rc) return rc;
    std::memset(info, 0, sizeof(*info));
    info->path = choose_path(c);
    c.ldg = info->path == HARRIS_PATH_LDG;
    c.pair = info->path == HARRIS_PATH_PAIR || info->path == HARRIS_PATH_QUAD;
    c.group = info->path == HARRIS_PATH_QUAD ? 4 : 2;
    c.cfg = (c.ldg || c.pair) ? -1 : resolve_cfg(ctx, c);
    const TmaConfig& cfg = c.pair ? (c.group == 4 ? kQuadConfig : kPairConfig)
                           : c.ldg ? kLdgConfigs[ctx->ldg_cfg]
                                   : kTmaConfigs[c.cfg];
    info->warps_per_cta = cfg.warps;
    info->stages = cfg.stages;
    info->rows_per_stage = cfg.rows;
    TileGeom tg;
    int64_t grid = 0;
    plan_launch(ctx, c, tg, grid);
    info->band_rows = tg.band_rows;
    info->bands = tg.bands;
    info->col_segments = tg.colsegs;
    info->tiles = tg.tiles;
    info->grid_ctas = grid;
    info->smem_bytes = (c.ldg || c.pair) ? 0 : int64_t(tma_smem_bytes(c.cfg));
    info->groups = cfg.groups;
    info->tma_config = c.cfg;  // -1: the LDG kernel
    info->strip_cols = cfg.strip_cols;
    return HARRIS_OK;
}

int harris_last_path(const harris_ctx* ctx) { return ctx ? ctx->last_path.load() : HARRIS_PATH_NONE; }
int harris_device(const harris_ctx* ctx) { return ctx ? ctx->device : -1; }
int harris_num_sms(const harris_ctx* ctx) { return ctx ? ctx->num_sms : 0; }
const char* harris_last_cuda_error(const harris_ctx* ctx) { return ctx ? ctx->last_err : ""; }

int harris_synth_fill(float* dst, int64_t planes, int64_t rows, int64_t W, int64_t dst_pitch,
                      int64_t dst_plane_stride, int64_t H_global, int64_t row0, int64_t plane0, uint64_t seed,
                      int dist, void* stream) {
    if (!dst || planes < 0 || rows < 0 || W < 1 || dst_pitch < W || row0 < 0 || plane0 < 0 ||
        row0 + rows > H_global || (planes > 1 && dst_plane_stride < rows * dst_pitch))
        return HARRIS_ERR_INVALID_ARGUMENT;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = launch_synth(dst, planes, rows, W, dst_pitch, dst_plane_stride, H_global, row0, plane0, seed,
                                 dist, sms, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HARRIS_OK : HARRIS_ERR_CUDA;
}

int64_t harris_grouping_scratch_bytes(int grouping, int64_t n, int64_t m) {
    if (n < 1 || m < 1) return -1;
    const int64_t f = grouping_scratch_floats(grouping, n, m);
    if (f < 0) return -1;
    // enough for both implementations: the Appendix-B kernels (EXACT) and the strip-engine
    // kernels (FAST, 16-byte aligned plane pitches)
    return std::max(f, grouping_fast_scratch_floats(grouping, n, m)) * 4;
}

int harris_grouping_launches(int grouping) { return grouping_launches(grouping); }

int harris_run_grouping(harris_ctx* ctx, int grouping, float* out, int64_t n, int64_t m, const float* rgb,
                        void* scratch, int64_t scratch_bytes, float kappa, uint32_t flags, void* stream) {
    if (!ctx || !out || !rgb) return HARRIS_ERR_INVALID_ARGUMENT;
    if (n < 1 || m < 1) return HARRIS_ERR_SIZE;
    if (grouping == HARRIS_GROUPING_FUSED) {
        const int64_t W = m + 4, H = n + 4;
        return run(ctx, make_call(out, m, n * m, n, m, rgb, W, H * W, 3 * H * W, 1, kappa, flags),
                   static_cast<cudaStream_t>(stream));
    }
    const int64_t need = harris_grouping_scratch_bytes(grouping, n, m);
    if (need < 0) return HARRIS_ERR_INVALID_ARGUMENT;
    if (!scratch || scratch_bytes < need) return HARRIS_ERR_INVALID_ARGUMENT;
    DeviceGuard guard(ctx->device);
    if (!guard.ok) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
    // FAST (default): every group a strip-engine kernel in the fused kernel's arithmetic (the
    // fair ablation; needs the TMA layout: W % 4 == 0, 16-byte aligned rgb / scratch / out);
    // HARRIS_FLAG_EXACT_ORDER or other layouts: the Appendix-B one-thread-per-pixel kernels
    const bool fast = !(flags & HARRIS_FLAG_EXACT_ORDER) && ((m + 4) & 3) == 0 && aligned16(rgb) &&
                      aligned16(scratch) && aligned16(out) && (m & 3) == 0;
    if (fast) {
        const GroupLaunchEnv env{ctx->encode, ctx->num_sms, ctx->occ_grp, ctx->l2_policy};
        const int rc = launch_grouping_fast(env, grouping, out, n, m, rgb, static_cast<float*>(scratch), kappa,
                                            static_cast<cudaStream_t>(stream));
        if (rc < 0) {
            std::snprintf(ctx->last_err, sizeof(ctx->last_err), "cuTensorMapEncodeTiled (grouping) failed");
            return HARRIS_ERR_TMA;
        }
        if (rc) return cuda_fail(ctx, cudaGetLastError(), "launch grouping (fast)");
        ctx->last_path = HARRIS_PATH_TMA;
        return HARRIS_OK;
    }
    cudaError_t e = launch_grouping(grouping, out, n, m, rgb, static_cast<float*>(scratch), kappa, ctx->num_sms,
                                    static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch grouping");
    ctx->last_path = HARRIS_PATH_NONE;
    return HARRIS_OK;
}

// ------------------------------------------------------------- host buffers
static int ensure_staging(harris_ctx* ctx, size_t in_bytes, size_t out_bytes) {
    cudaError_t e;
    for (int k = 0; k < harris_ctx::kSlots; ++k) {
        if (!ctx->streams[k]) {
            e = cudaStreamCreateWithFlags(&ctx->streams[k], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamCreate");
        }
    }
    if (in_bytes > ctx->cap_in) {
        for (int k = 0; k < harris_ctx::kSlots; ++k) {
            cudaFree(ctx->d_in[k]);
            ctx->d_in[k] = nullptr;
            e = cudaMalloc(&ctx->d_in[k], in_bytes);
            if (e != cudaSuccess) {
                ctx->cap_in = 0;
                return cuda_fail(ctx, e, "cudaMalloc staging in");
            }
        }
        ctx->cap_in = in_bytes;
    }
    if (out_bytes > ctx->cap_out) {
        for (int k = 0; k < harris_ctx::kSlots; ++k) {
            cudaFree(ctx->d_out[k]);
            ctx->d_out[k] = nullptr;
            e = cudaMalloc(&ctx->d_out[k], out_bytes);
            if (e != cudaSuccess) {
                ctx->cap_out = 0;
                return cuda_fail(ctx, e, "cudaMalloc staging out");
            }
        }
        ctx->cap_out = out_bytes;
    }
    return HARRIS_OK;
}

static int run_host_impl(harris_ctx* ctx, int fmt, float* out_host, int64_t out_pitch, int64_t n, int64_t m,
                         const void* in_host, int64_t batch, float kappa, uint32_t flags) {
    if (!ctx || !out_host || !in_host) return HARRIS_ERR_INVALID_ARGUMENT;
    if (n < 1 || m < 1) return HARRIS_ERR_SIZE;
    if (batch < 1 || out_pitch < m) return HARRIS_ERR_INVALID_ARGUMENT;
    NvtxRange nvtx(fmt == kU8Interleaved ? "harris_run_host_u8" : "harris_run_host");
    DeviceGuard guard(ctx->device);
    if (!guard.ok) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
    const bool u8 = fmt == kU8Interleaved;
    const int64_t H = n + 4, W = m + 4;
    // bytes of one input row of all channels, and of one image
    const int64_t row_bytes = u8 ? 3 * W : 3 * W * 4;
    const int64_t img_bytes = H * row_bytes;
    const int64_t kChunkBytes = int64_t(48) << 20;  // input bytes per pipeline chunk
    // chunk = a group of whole images, or (batch == 1 and large) a row band + 4-row halo
    const bool banded = batch == 1 && img_bytes > kChunkBytes;
    const int64_t imgs_per_chunk = banded ? 1 : std::max<int64_t>(1, kChunkBytes / img_bytes);
    const int64_t band_rows = banded ? std::max<int64_t>(1, kChunkBytes / row_bytes - 4) : n;
    const size_t in_bytes = size_t(banded ? (band_rows + 4) * row_bytes : imgs_per_chunk * img_bytes);
    const size_t out_bytes = size_t(banded ? band_rows * m : imgs_per_chunk * n * m) * 4;
    int rc = ensure_staging(ctx, in_bytes, out_bytes);
    if (rc) return rc;
    const int64_t nchunks = banded ? (n + band_rows - 1) / band_rows : (batch + imgs_per_chunk - 1) / imgs_per_chunk;
    const unsigned char* src = static_cast<const unsigned char*>(in_host);
    cudaError_t e = cudaSuccess;
    for (int64_t k = 0; k < nchunks && rc == HARRIS_OK; ++k) {
        const int slot = int(k % harris_ctx::kSlots);
        cudaStream_t s = ctx->streams[slot];
        unsigned char* din = reinterpret_cast<unsigned char*>(ctx->d_in[slot]);
        float* dout = ctx->d_out[slot];
        int64_t rows = n, nb = 1, r0 = 0, b0 = 0;
        Call c;
        if (banded) {
            r0 = k * band_rows;
            rows = std::min(band_rows, n - r0);
            const int64_t rin = rows + 4;
            if (u8) {  // HWC: the band is one contiguous run of rows
                e = cudaMemcpyAsync(din, src + r0 * 3 * W, size_t(rin * 3 * W), cudaMemcpyHostToDevice, s);
                c = make_call(dout, m, rows * m, rows, m, reinterpret_cast<const float*>(din), 3 * W, 0,
                              rin * 3 * W, 1, kappa, flags);
            } else {   // planar: one run per channel
                for (int ch = 0; ch < 3 && e == cudaSuccess; ++ch)
                    e = cudaMemcpyAsync(din + size_t(ch * rin * W) * 4, src + size_t(ch * H * W + r0 * W) * 4,
                                        size_t(rin * W) * 4, cudaMemcpyHostToDevice, s);
                c = make_call(dout, m, rows * m, rows, m, reinterpret_cast<const float*>(din), W, rin * W,
                              3 * rin * W, 1, kappa, flags);
            }
            if (e != cudaSuccess) {  // stop issuing; the final sync below still drains every slot
                rc = cuda_fail(ctx, e, "H2D band");
                break;
            }
        } else {
            b0 = k * imgs_per_chunk;
            nb = std::min(imgs_per_chunk, batch - b0);
            e = cudaMemcpyAsync(din, src + size_t(b0 * img_bytes), size_t(nb * img_bytes), cudaMemcpyHostToDevice,
                                s);
            if (e != cudaSuccess) {  // stop issuing; the final sync below still drains every slot
                rc = cuda_fail(ctx, e, "H2D images");
                break;
            }
            c = u8 ? make_call(dout, m, n * m, n, m, reinterpret_cast<const float*>(din), 3 * W, 0, img_bytes, nb,
                               kappa, flags)
                   : make_call(dout, m, n * m, n, m, reinterpret_cast<const float*>(din), W, H * W, 3 * H * W, nb,
                               kappa, flags);
        }
        c.fmt = fmt;
        rc = run(ctx, c, s);
        if (rc) break;
        e = cudaMemcpy2DAsync(out_host + (banded ? r0 : b0 * n) * out_pitch, size_t(out_pitch) * 4, dout,
                              size_t(m) * 4, size_t(m) * 4, size_t(banded ? rows : nb * n), cudaMemcpyDeviceToHost,
                              s);
        if (e != cudaSuccess) {  // stop issuing; the final sync below still drains every slot
                rc = cuda_fail(ctx, e, "D2H");
                break;
            }
    }
    for (int k = 0; k < harris_ctx::kSlots; ++k) {
        cudaError_t se = cudaStreamSynchronize(ctx->streams[k]);
        if (se != cudaSuccess && rc == HARRIS_OK) rc = cuda_fail(ctx, se, "pipeline sync");
    }
    return rc;
}

int harris_run_host(harris_ctx* ctx, float* out_host, int64_t out_pitch, int64_t n, int64_t m,
                    const float* rgb_host, int64_t batch, float kappa, uint32_t flags) {
    return run_host_impl(ctx, kF32Planar, out_host, out_pitch, n, m, rgb_host, batch, kappa, flags);
}

int harris_run_host_u8(harris_ctx* ctx, float* out_host, int64_t out_pitch, int64_t n, int64_t m,
                       const uint8_t* rgb8_host, int64_t batch, float kappa, uint32_t flags) {
    return run_host_impl(ctx, kU8Interleaved, out_host, out_pitch, n, m, rgb8_host, batch, kappa, flags);
}

}  // extern "C"
