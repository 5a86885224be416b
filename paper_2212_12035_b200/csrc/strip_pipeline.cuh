// strip_pipeline.cuh — the warp-strip TMA engine shared by every fused stencil
// in this library (Harris f32, Harris u8-ingest, separable 3x3).
//
// Work decomposition: a *tile* is one 128-output-column warp strip x
// `band_rows` output rows of one image (TileGeom).  A persistent grid of
// NW-warp CTAs strides its warps over tiles; each warp runs its own pipeline (the
// only CTA-wide barrier is one named barrier per tile wave that keeps neighbouring
// strips in step for L2 halo reuse): it owns an NS-stage shared-memory ring, and its
// lane 0 issues one TMA box per stage (Op::load) completing on the stage's
// mbarrier.  The producer cursor runs NS stages ahead of the consumer and keeps
// going across tile boundaries, so the pipeline never drains between tiles.
//
// The consumer calls Op::row<R>() once per input row (R = row within the stage,
// a compile-time constant: the row loop is fully unrolled and the stage height
// is a multiple of the op's register-rotation period, so rolling-window state
// lives in registers with static slot indices — the thesis's register rotation,
// PAPER.md:4814-4815) and stores the 4 outputs of each lane once the window is
// full (input row i >= Op::kHaloRows).
//
// Op concept:
//   kGroups (1 or 2: strips per tile; with 2 a lane owns the same 4 columns of two
//            adjacent strips, so the op can run packed f32x2 math),
//   kStripCols (output columns per strip: 128, or 124 when lane 31 is the halo lane),
//   kRowsPerStage, kHaloRows, kStageBytes (multiple of 128), kTxBytes
//   struct Params;  explicit Op(const Params&)
//   static void load(void* smem, const CUtensorMap*, uint64_t* bar, const int (&strip_col0)[kGroups],
//                    int in_row0, const int (&image)[kGroups], uint64_t l2_policy)   // lane 0 only
//   template <int R> void row(const unsigned char* stage, int lane, float (&out)[kGroups][4])
#pragma once
#include <cuda.h>

#include <cstdint>
#include <type_traits>
#include <utility>

#include "harris_common.cuh"
#include "harris_internal.h"

namespace harris {

// Tile -> coordinates.  G = 1: tile t = (image b, band, strip cs), strip-fastest.
// G = 2: the strips of one band row of ALL images are numbered s = b * colsegs + cs and
// paired (2p, 2p+1), so a pair may straddle two images and no group idles at the
// right edge of an image; tile t = (band, pair p), pair-fastest.
template <int G>
struct TileCoord {
    int band;
    int b[G], cs[G];
    bool valid[G];
};

// 32-bit index math: the host guarantees tiles and batch * colsegs < 2^31 (tma_eligible),
// and a 32-bit divide is a fraction of the emulated 64-bit one
template <int G>
__device__ __forceinline__ TileCoord<G> decode_tile(int64_t t64, const TileGeom& g) {
    TileCoord<G> c;
    const uint32_t t = uint32_t(t64);
    if constexpr (G == 1) {
        const uint32_t q = t / uint32_t(g.colsegs);
        c.cs[0] = int(t - q * uint32_t(g.colsegs));
        const uint32_t b = q / uint32_t(g.bands);
        c.band = int(q - b * uint32_t(g.bands));
        c.b[0] = int(b);
        c.valid[0] = true;
    } else {
        const uint32_t strips = uint32_t(g.batch) * uint32_t(g.colsegs);
        const uint32_t pairs = (strips + 1) / 2;
        const uint32_t band = t / pairs;
        const uint32_t p = t - band * pairs;
        c.band = int(band);
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const uint32_t sidx = 2 * p + k;
            c.valid[k] = sidx < strips;
            const uint32_t s2 = c.valid[k] ? sidx : 0;
            const uint32_t b = s2 / uint32_t(g.colsegs);
            c.b[k] = int(b);
            c.cs[k] = int(s2 - b * uint32_t(g.colsegs));
        }
    }
    return c;
}

__device__ __forceinline__ int band_rows_out(int band, const TileGeom& g) {
    const int r = g.n - band * g.band_rows;
    return r < g.band_rows ? r : g.band_rows;
}

template <class F, int... Rs>
__device__ __forceinline__ void static_for(F&& f, std::integer_sequence<int, Rs...>) {
    (f(std::integral_constant<int, Rs>{}), ...);
}

// Op::kWarpLoad is optional (default false): the stage is filled by all 32 lanes with
// Op::load_warp(smem, params, bar, cols, row0, imgs, lane, l2_policy) (cp.async, for inputs TMA
// cannot describe) instead of one TMA issue by lane 0; the stage barrier then counts
// 32 arrivals instead of an expect_tx byte count
template <class Op, class = void>
struct WarpLoadOf : std::false_type {};
template <class Op>
struct WarpLoadOf<Op, std::void_t<decltype(Op::kWarpLoad)>> : std::integral_constant<bool, Op::kWarpLoad> {};

// Op::kBarArrivals is optional (warp loads only; default 32): arrivals per stage barrier
// phase — 1 for a warp load that issues bulk copies and one arrive.expect_tx
template <class Op, class = void>
struct BarArrivalsOf : std::integral_constant<int, 32> {};
template <class Op>
struct BarArrivalsOf<Op, std::void_t<decltype(Op::kBarArrivals)>> : std::integral_constant<int, Op::kBarArrivals> {};

// Op::kSplitStores is optional (default false): with true, output rows that are all 8-byte
// aligned but not 16-byte aligned (TileGeom::vec_store == 1, e.g. 1914-float rows) get two
// 8-byte stores per lane (fewer store transactions: +1.8 % on the pair-row kernel, whose
// outputs are typically that wide).  Off elsewhere: even the untaken second store variant
// in the unrolled row loop measured 23 % slower on the quad-row kernel (odd-width outputs,
// 404 -> 311 k) and 11 % on the issue-bound u8 kernels.
template <class Op, class = void>
struct SplitStoresOf : std::false_type {};
template <class Op>
struct SplitStoresOf<Op, std::void_t<decltype(Op::kSplitStores)>> : std::integral_constant<bool, Op::kSplitStores> {};

// Op::kRealignStores is optional (default false; single-strip ops): output rows that are only
// 8-byte aligned (TileGeom::vec_store == 1 — e.g. the 1918-float rows of a contiguous stencil
// output, whose rows alternate between 16- and 8-byte alignment) are written with 16-byte
// stores anyway: on a row that starts 8 bytes past a 16-byte boundary, lane L stores its last
// two outputs and lane L+1's first two (one shuffle pair) at the aligned address, lane 0 adds
// its first two and lane 31 its last two as 8-byte stores.  Rows that are 16-byte aligned keep
// one float4 per lane.  Replaces four scalar stores per lane per row.
template <class Op, class = void>
struct RealignStoresOf : std::false_type {};
template <class Op>
struct RealignStoresOf<Op, std::void_t<decltype(Op::kRealignStores)>>
    : std::integral_constant<bool, Op::kRealignStores> {};

// one output row of 4 values per lane at po (lane column cg of an m-column row whose start is
// 8-byte aligned); warp-uniform alignment test per row
__device__ __forceinline__ void stg_realigned_row(float* po, const float (&o)[4], int cg, int m, int lane) {
    const float n0 = __shfl_down_sync(0xffffffffu, o[0], 1);
    const float n1 = __shfl_down_sync(0xffffffffu, o[1], 1);
    if ((reinterpret_cast<uintptr_t>(po) & 15u) == 0) {
        if (cg + 4 <= m) {
            stg128_cs(po, o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (cg + k < m) po[k] = o[k];
        }
        return;
    }
    if (lane == 0) {
        if (cg + 2 <= m)
            stg64_cs(po, o[0], o[1]);
        else if (cg < m)
            po[0] = o[0];
    }
    if (lane < 31) {
        if (cg + 6 <= m) {
            stg128_cs(po + 2, o[2], o[3], n0, n1);
        } else {
            const float v[4] = {o[2], o[3], n0, n1};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (cg + 2 + k < m) po[2 + k] = v[k];
        }
    } else {
        if (cg + 4 <= m) {
            stg64_cs(po + 2, o[2], o[3]);
        } else if (cg + 2 < m) {
            po[2] = o[2];
        }
    }
}

// Op::kOutPlanes is optional (default 1; single-strip ops only): the op produces that many
// output planes per row (out[kOutPlanes][4]), stored at TileGeom::out_plane_stride apart —
// the unfused kernel groupings of the fusion ablation write Ix/Iy or the three products
template <class Op, class = void>
struct OutPlanesOf : std::integral_constant<int, 1> {};
template <class Op>
struct OutPlanesOf<Op, std::void_t<decltype(Op::kOutPlanes)>> : std::integral_constant<int, Op::kOutPlanes> {};

// Op::kTwoStoreVariants is optional (default false): compile the consumer's stage loop twice,
// with and without the scalar-store code for ragged / unaligned output lanes.  Measured per
// op (tools/perf_matrix.sh): issue-bound u8 TMA 840 -> 887 k MP/s, stencil on 1918-wide
// planes 727 -> 763 k; but the f32 TMA op -1.8 % and the u8 row-group op -4 % (code size)
template <class Op, class = void>
struct TwoStoreVariantsOf : std::false_type {};
template <class Op>
struct TwoStoreVariantsOf<Op, std::void_t<decltype(Op::kTwoStoreVariants)>>
    : std::integral_constant<bool, Op::kTwoStoreVariants> {};

// Op::load_p(smem, tmap, bar, cols, row0, imgs, policy, params) is optional: a TMA stage fill
// that needs the kernel parameters (the pair-row op's odd-row column offset)
template <class Op, class = void>
struct HasLoadP : std::false_type {};
template <class Op>
struct HasLoadP<Op, std::void_t<decltype(&Op::load_p)>> : std::true_type {};

// Op::kCacheProducer is optional (default true): decode the producer's tile once per tile
template <class Op, class = void>
struct CacheProducerOf : std::true_type {};
template <class Op>
struct CacheProducerOf<Op, std::void_t<decltype(Op::kCacheProducer)>>
    : std::integral_constant<bool, Op::kCacheProducer> {};

// Op::begin_tile(strip_col0, row0, image) is optional: per-tile state of the op (e.g. the
// u8 box skew)
template <class Op, class = void>
struct HasBeginTile : std::false_type {};
template <class Op>
struct HasBeginTile<Op, std::void_t<decltype(&Op::begin_tile)>> : std::true_type {};

// Op::kTmaStore is optional (default false): outputs leave through TMA stores instead of
// per-lane st.global.  Each warp owns two output staging buffers of kRowsPerStage x 128
// floats (Op::kOutStageBytes); the lanes write a stage's output rows there (st.shared.v4),
// fence them into the async proxy, and lane 0 stores them as 128 x 2-row boxes through the
// output tensor map Op::out_tmap(params) (cp.async.bulk.tensor, one bulk group per stage)
// while the warp computes the next stage into the other buffer.  The tensor map clips the
// right / bottom edges; band_rows must be even (a row pair never straddles two tiles).
// Single-strip ops (kGroups == 1, 128-column strips) only.
template <class Op, class = void>
struct TmaStoreOf : std::false_type {};
template <class Op>
struct TmaStoreOf<Op, std::void_t<decltype(Op::kTmaStore)>> : std::integral_constant<bool, Op::kTmaStore> {};

template <class Op, bool TS = TmaStoreOf<Op>::value>
struct OutStageBytesOf : std::integral_constant<size_t, 0> {};
template <class Op>
struct OutStageBytesOf<Op, true> : std::integral_constant<size_t, Op::kOutStageBytes> {};

template <int NW, int NS, class Op>
struct StripShape {
    static_assert(Op::kStageBytes % 128 == 0, "TMA destinations must be 128-byte aligned");
    static constexpr size_t kOutBytes = size_t(NW) * 2 * OutStageBytesOf<Op>::value;  // TMA-store staging
    static constexpr size_t kSmemBytes = size_t(NW) * NS * Op::kStageBytes + kOutBytes + size_t(NW) * NS * 8 + 128;
};

// Completion notification for fused gathers (TileGeom::notify_flag): every thread
// fences its output stores at system scope (they may be NVLink stores into a peer's
// buffer), the CTA meets at a barrier, and the last CTA to count itself in resets the
// counter and releases the epoch into the flag — the consumer on the other GPU acquires
// it (harris_peer_wait) and then sees every output row of this launch.
__device__ __forceinline__ void notify_epilogue(const TileGeom& g) {
    if (g.notify_flag == nullptr) return;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned done = atomicAdd(g.notify_counter, 1u);
        if (done == gridDim.x - 1) {
            __threadfence_system();  // acquire side of the other CTAs' fence + count
            *reinterpret_cast<volatile uint32_t*>(g.notify_counter) = 0u;
            st_release_sys(g.notify_flag, g.notify_epoch);
        }
    }
}

// Host-side launch of a strip kernel, with programmatic dependent launch when pdl != 0
// (cudaLaunchAttributeProgrammaticStreamSerialization): the kernel may start while the previous
// kernel on the stream is still running; it releases its own dependents at entry
// (griddepcontrol.launch_dependents) and, with pdl == 1, waits for the previous grid
// (griddepcontrol.wait) before its first global-memory access.
template <class Kern, class... Args>
inline cudaError_t launch_strip(Kern kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, int pdl,
                                const Args&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <class Op, int NW, int NS, int MINB = 1>
__global__ void __launch_bounds__(NW * 32, MINB)
    strip_kernel(const __grid_constant__ CUtensorMap tmap, const TileGeom g,
                 const __grid_constant__ typename Op::Params p) {
    constexpr int CH = Op::kRowsPerStage;
    constexpr int HALO = Op::kHaloRows;
    constexpr int G = Op::kGroups;
    constexpr int NP = OutPlanesOf<Op>::value;
    static_assert(NP == 1 || G == 1, "multi-plane outputs: single-strip ops");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // align by offsetting the __shared__ array itself (an integer round trip would turn
    // every stage read into a generic LD instead of LDS)
    unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned char* ring = base + size_t(warp) * NS * Op::kStageBytes;
    constexpr bool TS = TmaStoreOf<Op>::value;
    constexpr size_t kOutStage = OutStageBytesOf<Op>::value;
    static_assert(!TS || (G == 1 && Op::kStripCols == kWarpCols && CH % 2 == 0 && HALO % 2 == 0 &&
                          kOutStage == size_t(CH) * kWarpCols * 4 && kOutStage % 128 == 0),
                  "TMA-store ops: one 128-column strip, row pairs aligned with the stage and the halo");
    unsigned char* ostage = base + size_t(NW) * NS * Op::kStageBytes + size_t(warp) * 2 * kOutStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + size_t(NW) * NS * Op::kStageBytes +
                                                 StripShape<NW, NS, Op>::kOutBytes) + warp * NS;

    const int64_t GW = int64_t(gridDim.x) * NW;
    const int64_t gw = int64_t(blockIdx.x) * NW + warp;
    const int64_t cta0 = int64_t(blockIdx.x) * NW;  // first warp-tile index of this CTA
    // PDL (TileGeom::pdl).  Mode 2 (independent): release the next kernel at once — its CTAs
    // take the SMs this grid leaves — and let CTA 0 wait for the PREVIOUS grid before exiting,
    // so this grid still completes after everything before it (stream order for later work).
    // Mode 1: wait for the previous grid before the first global access (below), then release.
    if (g.pdl == 2) pdl_launch_dependents();
    if (cta0 >= g.tiles) {                          // whole CTA idle
        if (g.pdl == 1) {
            pdl_wait();
            pdl_launch_dependents();
        }
        notify_epilogue(g);
        if (g.pdl == 2 && blockIdx.x == 0) pdl_wait();
        return;
    }
    // waves in which at least one warp of this CTA has a tile: every warp of the CTA runs
    // this many wave iterations so the per-wave CTA barrier below is uniform
    const int64_t waves = (g.tiles - cta0 + GW - 1) / GW;

    constexpr bool kWarpLoad = WarpLoadOf<Op>::value;
    if (lane == 0) {
        if constexpr (!kWarpLoad) prefetch_tmap(&tmap);
#pragma unroll
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], kWarpLoad ? BarArrivalsOf<Op>::value : 1);
        fence_barrier_init();
    }
    __syncwarp();
    const uint64_t policy = l2_policy(g.l2_policy);

    // ---- producer cursor (warp-uniform; lane 0 issues).  With kCacheProducer the tile is
    // decoded once per tile instead of once per stage issue: fewer instructions on the
    // issue path (u8: +6-9 %, small images 18.5 -> 16.4 us), but for the f32 dual-strip op
    // the per-stage form measured 2-3 % faster (profiles/ab_producer_decode_r01.txt), so
    // the op opts out. ----
    constexpr bool kCacheP = CacheProducerOf<Op>::value;
    static_assert(!kWarpLoad || kCacheP, "warp loads use the cached producer tile");
    int64_t pt = gw;
    int pc = 0, pn = 0, prow0 = 0;
    int pcols[G], pimgs[G];
    auto decode_producer = [&]() {
        const TileCoord<G> c = decode_tile<G>(pt, g);
#pragma unroll
        for (int k = 0; k < G; ++k) {
            pcols[k] = c.cs[k] * Op::kStripCols;
            pimgs[k] = c.b[k];
        }
        prow0 = c.band * g.band_rows;
        pn = (band_rows_out(c.band, g) + HALO + CH - 1) / CH;
    };
    if constexpr (kCacheP) {
        if (pt < g.tiles) decode_producer();
    } else {
        pn = (band_rows_out(decode_tile<G>(pt, g).band, g) + HALO + CH - 1) / CH;
    }
    auto issue = [&](int s) {
        if (pt < g.tiles) {
            if constexpr (kWarpLoad) {
                Op::load_warp(ring + s * Op::kStageBytes, p, &bars[s], pcols, prow0 + pc * CH, pimgs, lane, policy);
            } else if (lane == 0) {
                if constexpr (kCacheP) {
                    mbar_arrive_expect_tx(&bars[s], Op::kTxBytes);
                    if constexpr (HasLoadP<Op>::value)
                        Op::load_p(ring + s * Op::kStageBytes, &tmap, &bars[s], pcols, prow0 + pc * CH, pimgs,
                                   policy, p);
                    else
                        Op::load(ring + s * Op::kStageBytes, &tmap, &bars[s], pcols, prow0 + pc * CH, pimgs,
                                 policy);
                } else {
                    const TileCoord<G> c = decode_tile<G>(pt, g);
                    int cols[G], imgs[G];
#pragma unroll
                    for (int k = 0; k < G; ++k) {
                        cols[k] = c.cs[k] * Op::kStripCols;
                        imgs[k] = c.b[k];
                    }
                    mbar_arrive_expect_tx(&bars[s], Op::kTxBytes);
                    Op::load(ring + s * Op::kStageBytes, &tmap, &bars[s], cols, c.band * g.band_rows + pc * CH,
                             imgs, policy);
                }
            }
            if (++pc == pn) {
                pc = 0;
                pt += GW;
                if (pt < g.tiles) {
                    if constexpr (kCacheP)
                        decode_producer();
                    else
                        pn = (band_rows_out(decode_tile<G>(pt, g).band, g) + HALO + CH - 1) / CH;
                }
            }
        }
    };
    // PDL mode 1: the prologue above (barrier init, tensor-map prefetch, first tile decode)
    // overlapped the previous kernel; memory is only touched after it completed
    if (g.pdl == 1) {
        pdl_wait();
        pdl_launch_dependents();
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) issue(s);

    Op op(p);
    int stage = 0;
    uint32_t phase = 0;
    int obuf = 0;  // TMA-store ops: staging buffer of the current stage
    (void)obuf;
    (void)ostage;
    for (int64_t k = 0; k < waves; ++k) {
        const int64_t t = gw + k * GW;
        // Re-align the CTA's warps at every tile boundary.  They work on adjacent strips
        // of the same band, whose 4-column halo sectors hit in L2 only while the warps
        // stay within a few microseconds of each other; without this the highest-wid-first
        // warp arbiter lets them drift apart over the waves and the halo re-reads miss
        // (DRAM read over-fetch 2-6.5 % -> measured in profiles/ncu_configs_r01.json).
        if (k > 0 && g.sync_waves) asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
        if (t >= g.tiles) continue;
        const TileCoord<G> tc = decode_tile<G>(t, g);
        const int rows_out = band_rows_out(tc.band, g);
        const int nch = (rows_out + HALO + CH - 1) / CH;
        if constexpr (HasBeginTile<Op>::value) {
            int c0[G], im[G];
#pragma unroll
            for (int k = 0; k < G; ++k) {
                c0[k] = tc.cs[k] * Op::kStripCols;
                im[k] = tc.b[k];
            }
            op.begin_tile(c0, tc.band * g.band_rows, im);
        }
        if constexpr (TS) {
            // ---- TMA-store stage loop: outputs go to the staging buffer, lane 0 stores row pairs
            const int ox = tc.cs[0] * kWarpCols, oy0 = tc.band * g.band_rows, oz = tc.b[0];
            const void* otm = Op::out_tmap(p);
            for (int c = 0; c < nch; ++c) {
                mbar_wait(&bars[stage], phase);
                const unsigned char* sm = ring + stage * Op::kStageBytes;
                float* so = reinterpret_cast<float*>(ostage + obuf * kOutStage);
                // the buffer's previous bulk group (two stages ago) must have finished reading it
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                static_for(
                    [&](auto rc) {
                        constexpr int R = decltype(rc)::value;
                        float out4[1][4];
                        op.template row<R>(sm, lane, out4);
                        sts128(so + R * kWarpCols + lane * kColsPerLane, out4[0][0], out4[0][1], out4[0][2],
                               out4[0][3]);
                    },
                    std::make_integer_sequence<int, CH>{});
                fence_proxy_async_shared();
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int q = 0; q < CH / 2; ++q) {
                        const int o = c * CH + 2 * q - HALO;  // first output row of the pair (tile-relative)
                        if (o >= 0 && o < rows_out) tma_store_3d(otm, so + 2 * q * kWarpCols, ox, oy0 + o, oz);
                    }
                    bulk_commit();
                }
                issue(stage);
                obuf ^= 1;
                if (++stage == NS) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            continue;
        }
        int colg[G];
        float* orow[G];
#pragma unroll
        for (int k = 0; k < G; ++k) {
            // invalid strip, or the halo lane of a 124-column strip: never stored
            const bool own = tc.valid[k] && lane * kColsPerLane < Op::kStripCols;
            colg[k] = own ? tc.cs[k] * Op::kStripCols + lane * kColsPerLane : g.m;
            orow[k] = g.out + int64_t(tc.b[k]) * g.out_image_stride +
                      int64_t(tc.band) * g.band_rows * g.out_pitch + (colg[k] < g.m ? colg[k] : 0);
        }
        // store mode per lane and group, fixed for the tile: a predicated 16-byte store, plus a
        // scalar path behind a warp-uniform branch for tiles with a ragged / unaligned lane
        bool vec[G];
        bool ragged = false;
#pragma unroll
        for (int k = 0; k < G; ++k) {
            vec[k] = g.vec_store == 2 && colg[k] + kColsPerLane <= g.m;
            ragged |= !vec[k] && colg[k] < g.m;
        }
        ragged = __any_sync(0xffffffffu, ragged);

        // the stage loop (a macro so that ops with Op::kTwoStoreVariants get it twice — tiles
        // without ragged / unaligned output lanes then carry no scalar-store code — while every
        // other op keeps the single runtime-tested copy: a lambda wrapper alone changed their
        // code generation, -4.5 % on the u8 row-group op)
#define HARRIS_STAGE_LOOP(RAGGED)                                                                                \
    for (int c = 0; c < nch; ++c) {                                                                              \
        mbar_wait(&bars[stage], phase);                                                                          \
        const unsigned char* sm = ring + stage * Op::kStageBytes;                                                \
        static_for(                                                                                              \
            [&](auto rc) {                                                                                       \
                constexpr int R = decltype(rc)::value;                                                           \
                const int i = c * CH + R; /* input row within the tile */                                        \
                float out4[G * NP][4];                                                                           \
                op.template row<R>(sm, lane, out4);                                                              \
                if (i >= HALO && i - HALO < rows_out) {                                                          \
                    _Pragma("unroll") for (int gp = 0; gp < G * NP; ++gp) {                                      \
                        /* NP > 1: output planes of one strip (G == 1) at out_plane_stride */                   \
                        const int gi = NP > 1 ? 0 : gp;                                                          \
                        float* po = orow[gi] + int64_t(i - HALO) * g.out_pitch +                                 \
                                    (NP > 1 ? int64_t(gp) * g.out_plane_stride : 0);                             \
                        stg128_cs_if(vec[gi], po, out4[gp][0], out4[gp][1], out4[gp][2], out4[gp][3]);           \
                        if (RAGGED) { /* unaligned output rows, or the ragged right edge */                      \
                            const int cg = colg[gi];                                                             \
                            if (RealignStoresOf<Op>::value && g.vec_store == 1) {                                \
                                stg_realigned_row(po, out4[gp], cg, g.m, lane);                                  \
                            } else if (!vec[gi] && cg < g.m) {                                                   \
                                if (SplitStoresOf<Op>::value && g.vec_store == 1 && cg + kColsPerLane <= g.m) {  \
                                    stg2x2_cs(po, out4[gp][0], out4[gp][1], out4[gp][2], out4[gp][3]);           \
                                } else {                                                                         \
                                    _Pragma("unroll") for (int k = 0; k < kColsPerLane; ++k) if (cg + k < g.m)   \
                                        po[k] = out4[gp][k];                                                     \
                                }                                                                                \
                            }                                                                                    \
                        }                                                                                        \
                    }                                                                                            \
                }                                                                                                \
            },                                                                                                   \
            std::make_integer_sequence<int, CH>{});                                                              \
        __syncwarp(); /* every lane is done with this stage: refill it */                                        \
        issue(stage);                                                                                            \
        if (++stage == NS) {                                                                                     \
            stage = 0;                                                                                           \
            phase ^= 1u;                                                                                         \
        }                                                                                                        \
    }
        if constexpr (TwoStoreVariantsOf<Op>::value) {
            if (ragged) {
                HARRIS_STAGE_LOOP(true)
            } else {
                HARRIS_STAGE_LOOP(false)
            }
        } else {
            HARRIS_STAGE_LOOP(ragged)
        }
#undef HARRIS_STAGE_LOOP
    }
    if constexpr (TS) {
        if (lane == 0) bulk_wait_all();  // every TMA store performed (and its staging read) before exit
    }
    notify_epilogue(g);
    if (g.pdl == 2 && blockIdx.x == 0) pdl_wait();  // complete only after the previous grid
}

}  // namespace harris
