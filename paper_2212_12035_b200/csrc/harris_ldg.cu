// harris_ldg.cu — the fused Harris strip engine for inputs TMA cannot describe.
//
// TMA needs 16-byte aligned row starts and strides; a planar image whose rows are not
// 16-byte multiples (and not served by the pair- / quad-row tensor maps), a column-crop
// view whose base is only 4-byte aligned, or interleaved u8 rows of arbitrary byte pitch
// have neither.  Such inputs used to fall back to the generic shared-memory tile kernel
// K0 (118 k MP/s, 29 % of HBM).  The ops here keep everything of the TMA path — the
// warp-strip pipeline, the cores, the stage ring and its mbarriers — and only replace the
// stage fill, in two ways:
//  * K1b (default): one `cp.async.bulk` per stage row, issued by its own lane, counted as
//    transaction bytes on the stage mbarrier like a TMA box (F32BulkOp, U8BulkOp,
//    SepBulkOp; bulk_stage_fill).  The consumer reads each row at its skew from the
//    16-byte aligned-down copy start.
//  * K2: all 32 lanes copy the stage with 4-byte (u8: 4/16-byte) cp.async (LDGSTS) into the
//    TMA box's shared-memory layout, each lane's `cp.async.mbarrier.arrive.noinc`
//    completing the stage barrier (LdgOp, U8LdgOp; HARRIS_LDG_CONFIG 0-2,
//    HARRIS_U8LDG_CHUNK 4/16).
// Rows beyond the image are skipped and columns beyond the row end are stale or
// zero-filled; neither reaches a stored output.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "harris_common.cuh"
#include "harris_internal.h"
#include "harris_ops.cuh"
#include "harris_ops2.cuh"
#include "stencil_sep.cuh"
#include "strip_pipeline.cuh"

namespace harris {

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}

// one box row of kBoxCols floats, chunked by the row's own alignment (warp-uniform: the
// strip starts at a multiple of 128 columns): 16-byte copies for 16-byte aligned rows,
// 8-byte for 8-byte aligned ones, 4-byte otherwise; columns at or beyond `avail` are
// zero-filled (src-size 0 reads nothing)
template <int BYTES, int ROW = kBoxCols>
__device__ __forceinline__ void copy_row(float* dst, const float* src, int avail, int lane) {
    constexpr int E = BYTES / 4;                          // floats per chunk
    constexpr int NCH = (ROW + E - 1) / E;                // chunks per row
#pragma unroll
    for (int j = lane; j < NCH; j += 32) {
        const int c0 = j * E;
        const int valid = avail - c0;                     // floats of this chunk inside the row
        const uint32_t nb = valid >= E ? uint32_t(BYTES) : valid > 0 ? uint32_t(valid) * 4u : 0u;
        const float* sp = src + (nb ? c0 : 0);
        if constexpr (BYTES == 16)
            cp_async16(dst + c0, sp, nb);
        else if constexpr (BYTES == 8)
            cp_async8(dst + c0, sp, nb);
        else
            cp_async4(dst + c0, sp, nb);
    }
}

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// BYTES: copy granularity (4; wider copies measured slower: per-row 16/8/4 selection
// -27 %, 8-byte on 8-byte aligned rows -7 %, profiles/ab_ldg_r01.txt).  BaseOp: the TMA
// path's op whose shared-memory box layout and row arithmetic are reused unchanged.
// planes per input image (3 for the Harris ops, 1 for the separable stencil) and the
// shared-memory row width of the base op's box
template <class Op, class = void>
struct PlanesOf : std::integral_constant<int, 3> {};
template <class Op>
struct PlanesOf<Op, std::void_t<decltype(Op::kPlanes)>> : std::integral_constant<int, Op::kPlanes> {};
template <class Op, class = void>
struct BoxFloatsOf : std::integral_constant<int, kBoxCols> {};
template <class Op>
struct BoxFloatsOf<Op, std::void_t<decltype(Op::kBox)>> : std::integral_constant<int, Op::kBox> {};

template <class BaseOp, int BYTES>
struct LdgOp : BaseOp {
    static constexpr int G = BaseOp::kGroups;
    static constexpr int CH = BaseOp::kRowsPerStage;
    static constexpr int P = PlanesOf<BaseOp>::value;
    static constexpr int kRowFloats = BoxFloatsOf<BaseOp>::value;  // 132, or 128 in the lane-halo layout
    // byte distance between the G boxes of a stage (the TMA layout): P planes x CH rows,
    // padded to 128 bytes
    static constexpr uint32_t kBoxBytes = (uint32_t(P) * CH * kRowFloats * 4u + 127u) / 128u * 128u;
    static constexpr bool kWarpLoad = true;
    static constexpr bool kCacheProducer = true;
    struct Params {
        typename BaseOp::Params base;
        const float* src;
        int64_t in_pitch, in_plane_stride, in_image_stride;  // elements
        int32_t W, H;                                        // input columns / rows per image
        const void* limit;  // one past the view's last element (used by the bulk-copy ops)
    };

    __device__ __forceinline__ explicit LdgOp(const Params& p) : BaseOp(p.base) {}

    __device__ __forceinline__ static void load_warp(void* smem, const Params& p, uint64_t* bar,
                                                     const int (&col0)[G], int row0, const int (&image)[G],
                                                     int lane, uint64_t policy) {
        unsigned char* s = static_cast<unsigned char*>(smem);
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const float* img = p.src + int64_t(image[k]) * p.in_image_stride + col0[k];
            const int avail = p.W - col0[k];  // columns of this row from col0 to the row end
#pragma unroll
            for (int ch = 0; ch < P; ++ch) {
#pragma unroll
                for (int r = 0; r < CH; ++r) {
                    const int y = row0 + r;
                    if (y >= p.H) continue;  // below the image: never reaches a stored output
                    const float* src = img + int64_t(ch) * p.in_plane_stride + int64_t(y) * p.in_pitch;
                    float* dst = reinterpret_cast<float*>(s + k * kBoxBytes) + (ch * CH + r) * kRowFloats;
                    copy_row<BYTES, kRowFloats>(dst, src, avail, lane);
                }
            }
        }
        cp_async_mbar_arrive_noinc(bar);
    }
};

// HINT: an L2 cache-policy hint like the TMA input loads (`policy`: the kernel's createpolicy
// value of the ctx's l2_policy, evict_last by default, whose halo sectors are re-read by the
// neighbouring strip): +2 % on memory-bound
// f32 planes, -1 % on the issue-bound u8 / stencil ops (the extra createpolicy), so only
// F32BulkOp asks for it
template <bool HINT = false>
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy = 0) {
    if constexpr (HINT) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
            "%4;" ::"r"(smem_u32(smem)),
            "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
            : "memory");
    } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(smem)),
                     "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
                     : "memory");
    }
}

// The stage fill of the bulk-copy ops: each active lane copies one stage row — the bytes
// [src, src + need) (need: to the row end, capped by the slot) — as ONE bulk copy from the
// 16-byte aligned-down start, rounded up to whole 16-byte blocks.  Where that rounding would
// read past the view's last byte (`limit`; only an image's last row can reach it, flagged
// by `last_row`, so the test stays off every other row's path), the bulk part stops at the
// last whole block and the lane copies the < 16-byte tail itself with plain loads and
// shared stores, so no byte outside the view is ever read (compute-sanitizer memcheck
// clean with exact-size allocations).  The warp then syncs (ordering the tail stores before
// lane 0's release) and lane 0 arms the barrier with the warp's bulk bytes.
constexpr int kBulkBarArrivals = 1;
// cold path of bulk_stage_fill, out of line so the stage-fill path stays straight-line:
// shrink the bulk part to the whole 16-byte blocks before `limit` and copy the rest of the
// view's last bytes with plain loads / shared stores; returns the new bulk size
__device__ __noinline__ uint32_t bulk_tail_fix(unsigned char* dst, const unsigned char* al, const void* limit,
                                               uint32_t nb) {
    const uintptr_t room = reinterpret_cast<uintptr_t>(limit) - reinterpret_cast<uintptr_t>(al);
    if (room >= nb) return nb;
    const uint32_t whole = uint32_t(room) & ~15u;
    for (uint32_t i = whole; i < uint32_t(room); ++i) {
        uint32_t v;
        asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(al + i));
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(smem_u32(dst + i)), "r"(v));
    }
    return whole;
}

// STRICT (chosen by the host only when the view's end is not 16-byte aligned, i.e. when the
// rounding can reach past it): the stage that holds an image's last row (warp-uniform test)
// sends that row's lane through bulk_tail_fix.  A separate instantiation because even the
// untaken test measured 2-6 % slower on every other stage.
template <bool STRICT, bool HINT = false>
__device__ __forceinline__ void bulk_stage_fill(unsigned char* dst, const void* src, uint32_t need, uint32_t cap,
                                                const void* limit, uint64_t* bar, bool active,
                                                bool stage_has_last_row, bool last_row, int lane,
                                                uint64_t policy = 0) {
    uint32_t nb = 0;
    const unsigned char* al = nullptr;
    if (active) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(src);
        al = reinterpret_cast<const unsigned char*>(a & ~uintptr_t(15));
        const uint32_t up0 = (uint32_t(a & 15u) + need + 15u) & ~15u;
        nb = up0 < cap ? up0 : cap;
    }
    if constexpr (STRICT) {
        if (stage_has_last_row && active && last_row) nb = bulk_tail_fix(dst, al, limit, nb);
    }
    const uint32_t total = __reduce_add_sync(0xffffffffu, nb);
    if constexpr (STRICT) __syncwarp();  // the tail's shared stores before lane 0's release
    if (lane == 0) mbar_arrive_expect_tx(bar, total);
    __syncwarp();
    if (nb) bulk_g2s<HINT>(dst, al, nb, bar, policy);
}

// ---- planar f32 through the bulk-copy engine (K1b): every (channel, row) of a stage is
// ONE cp.async.bulk of <= 544 bytes from the row's 16-byte aligned-down start, issued by
// its own lane (G * 3 * CH <= 32 copies: the stage fill is one warp instruction), counted
// as transaction bytes on the stage mbarrier.  The consumer reads each lane's 4 floats
// at the row's float skew s (0..3; per strip and channel, advancing by pitch mod 4 per
// row): s even -> two 8-byte loads, s odd -> scalar + 8-byte + scalar, then the unchanged
// TMA-path core (no row-pair sums: FAST bit-identical to every other f32 path).
template <bool EXACT, int CH, int G, bool STRICT = false>
struct F32BulkOp : std::conditional_t<G == 2, HarrisF32x2Op<EXACT, CH, 124>, HarrisF32Op<EXACT, CH, 124>> {
    using Base = std::conditional_t<G == 2, HarrisF32x2Op<EXACT, CH, 124>, HarrisF32Op<EXACT, CH, 124>>;
    static_assert(G * 3 * CH <= 32, "one lane per stage row");
    static constexpr bool kWarpLoad = true;
    static constexpr int kBarArrivals = kBulkBarArrivals;
    static constexpr bool kCacheProducer = true;
    static constexpr int kRowFloats = 136;  // 544 B >= 3 skew floats + 128 columns, 16-byte multiple
    static constexpr uint32_t kBoxBytes = 3u * CH * kRowFloats * 4u;
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kStageBytes = uint32_t(G) * kBoxStride;
    struct Params {
        typename Base::Params base;
        const float* src;
        int64_t in_pitch, in_plane_stride, in_image_stride;  // elements
        int32_t W, H;                                        // input columns / rows per image
        const void* limit;                                   // one past the view's last element
    };
    uint32_t base_r, pitch_r, plane_r, image_r;  // float-index residues mod 4
    uint32_t sk[G][3];                           // current row's skew per strip and channel

    __device__ __forceinline__ explicit F32BulkOp(const Params& p)
        : Base(p.base),
          base_r(uint32_t(reinterpret_cast<uintptr_t>(p.src) >> 2) & 3u),
          pitch_r(uint32_t(p.in_pitch) & 3u),
          plane_r(uint32_t(p.in_plane_stride) & 3u),
          image_r(uint32_t(p.in_image_stride) & 3u) {}

    __device__ __forceinline__ void begin_tile(const int (&col0)[G], int row0, const int (&image)[G]) {
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const uint32_t s = base_r + uint32_t(image[k]) * image_r + uint32_t(row0) * pitch_r + uint32_t(col0[k]);
#pragma unroll
            for (int c = 0; c < 3; ++c) sk[k][c] = (s + uint32_t(c) * plane_r) & 3u;
        }
    }

    __device__ __forceinline__ static void load_warp(void* smem, const Params& p, uint64_t* bar,
                                                     const int (&col0)[G], int row0, const int (&image)[G],
                                                     int lane, uint64_t policy) {
        const int k = lane >= 3 * CH ? 1 : 0, rem = lane - k * 3 * CH;
        const int ch = rem / CH, r = rem - ch * CH;
        const int y = row0 + r;
        const int img = k ? image[G - 1] : image[0], c0 = k ? col0[G - 1] : col0[0];  // selects: no local array
        const float* src =
            p.src + int64_t(img) * p.in_image_stride + int64_t(ch) * p.in_plane_stride + int64_t(y) * p.in_pitch + c0;
        bulk_stage_fill<STRICT, true>(
            static_cast<unsigned char*>(smem) + k * kBoxStride + (ch * CH + r) * (kRowFloats * 4), src,
            uint32_t(p.W - c0) * 4u, kRowFloats * 4, p.limit, bar, lane < G * 3 * CH && y < p.H,
            row0 + CH > p.H - 1 && row0 <= p.H - 1, y == p.H - 1, lane, policy);
    }

    // 4 floats at q + s (q 16-byte aligned, s warp-uniform in 0..3)
    __device__ __forceinline__ static void read4(const float* q, uint32_t s, float (&c)[4]) {
        if (s & 1u) {
            const float2 v = lds64(q + s + 1);
            c[0] = q[s], c[1] = v.x, c[2] = v.y, c[3] = q[s + 3];
        } else {
            const float2 v0 = lds64(q + s), v1 = lds64(q + s + 2);
            c[0] = v0.x, c[1] = v0.y, c[2] = v1.x, c[3] = v1.y;
        }
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[G][4]) {
        float v[G][3][4];
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const float* box = reinterpret_cast<const float*>(stage + k * kBoxStride);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                read4(box + (c * CH + R) * kRowFloats + 4 * lane, sk[k][c], v[k][c]);
                sk[k][c] = (sk[k][c] + pitch_r) & 3u;
            }
        }
        if constexpr (G == 2) {
            float2 gown[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                gown[i] = make_float2(gray_of<EXACT>(v[0][0][i], v[0][1][i], v[0][2][i]),
                                      gray_of<EXACT>(v[1][0][i], v[1][1][i], v[1][2][i]));
            this->core.template step<R>(gown, lane, NoHalo{}, out);
        } else {
            float gown[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) gown[i] = gray_of<EXACT>(v[0][0][i], v[0][1][i], v[0][2][i]);
            this->core.template step<R, NoHalo, false>(gown, lane, NoHalo{}, out[0]);
        }
    }
};

// ---- interleaved u8 (HWC) rows at any byte alignment.  TMA needs 16-byte row strides
// (3W % 16 == 0); other widths get 4-byte cp.async of the row's words from its 4-byte
// aligned-down start, and the consumer realigns each lane's 3 words with funnel shifts by
// the row's byte skew (a running value: the op sees the tile's rows in order).
// A: copy granularity in bytes (4: 4-byte copies from the 4-byte aligned-down start; 16:
// one 16-byte copy per lane per row from the 16-byte aligned-down start, the consumer
// then also skips skew / 4 whole words)
template <bool EXACT, int CH, int A>
struct U8LdgOp : HarrisU8Op<EXACT, CH, 124> {
    using Base = HarrisU8Op<EXACT, CH, 124>;
    static_assert(A == 4 || A == 16, "u8 K2 copy granularity");
    static constexpr bool kWarpLoad = true;
    static constexpr bool kCacheProducer = true;
    static constexpr int kRowWords = Base::kWords;  // 100 words: 96 of 128 px + up to 15 skew bytes
    static constexpr int kChunks = A == 4 ? 97 : 25;  // copies per row
    static constexpr uint32_t kMask = A - 1;
    struct Params {
        float kappa;
        const uint8_t* rgb;
        int64_t in_pitch, in_image_stride;  // bytes
        int32_t W, H;                       // input pixels per row / rows per image
    };
    uint32_t base_r, pitch_r, image_r;  // byte address residues mod A
    uint32_t skew = 0;                  // misalignment (bytes, mod A) of the current row's start

    __device__ __forceinline__ explicit U8LdgOp(const Params& p)
        : Base(typename Base::Params{p.kappa}),
          base_r(uint32_t(reinterpret_cast<uintptr_t>(p.rgb)) & kMask),
          pitch_r(uint32_t(p.in_pitch) & kMask),
          image_r(uint32_t(p.in_image_stride) & kMask) {}

    __device__ __forceinline__ void begin_tile(const int (&col0)[1], int row0, const int (&image)[1]) {
        skew = (base_r + uint32_t(image[0]) * image_r + uint32_t(row0) * pitch_r + uint32_t(col0[0]) * 3u) & kMask;
    }

    __device__ __forceinline__ static void load_warp(void* smem, const Params& p, uint64_t* bar,
                                                     const int (&col0)[1], int row0, const int (&image)[1],
                                                     int lane, uint64_t policy) {
        uint32_t* s = static_cast<uint32_t*>(smem);
        const uint8_t* img = p.rgb + int64_t(image[0]) * p.in_image_stride + int64_t(col0[0]) * 3;
        const int avail_px = p.W - col0[0];
#pragma unroll
        for (int r = 0; r < CH; ++r) {
            const int y = row0 + r;
            if (y >= p.H) continue;  // below the image: never reaches a stored output
            const uint8_t* src = img + int64_t(y) * p.in_pitch;
            const uintptr_t a = reinterpret_cast<uintptr_t>(src);
            const uint8_t* al = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(kMask));
            const int avail = int(a & kMask) + avail_px * 3;  // bytes from `al` to the row end
            uint32_t* dst = s + r * kRowWords;
#pragma unroll
            for (int j = lane; j < kChunks; j += 32) {
                const int v = avail - A * j;
                const uint32_t nb = v >= A ? uint32_t(A) : v > 0 ? uint32_t(v) : 0u;
                if constexpr (A == 16)
                    cp_async16(dst + 4 * j, al + (nb ? 16 * j : 0), nb);
                else
                    cp_async4(dst + j, al + (nb ? 4 * j : 0), nb);
            }
        }
        cp_async_mbar_arrive_noinc(bar);
    }

    template <int R, int RP = R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(stage) + R * kRowWords + (skew >> 2) + 3 * lane;
        const uint32_t sh = (skew & 3u) * 8u;
        const uint32_t w3 = w[3];
        const uint32_t a0 = __funnelshift_r(w[0], w[1], sh), a1 = __funnelshift_r(w[1], w[2], sh),
                       a2 = __funnelshift_r(w[2], w3, sh);
        float gown[4];
        gray4_u8<EXACT>(a0, a1, a2, gown[0], gown[1], gown[2], gown[3]);
        this->core.template step<R, NoHalo, (CH % 2 == 0)>(gown, lane, NoHalo{}, out[0]);
        skew = (skew + pitch_r) & kMask;
    }
};

// u8 rows at any byte alignment through the bulk-copy engine (K1b).  TMA tensor maps need
// 16-byte row strides, which an interleaved row of 3W bytes has only when W % 16 == 0; a
// plain bulk copy (cp.async.bulk, no tensor map) needs only a 16-byte aligned source and
// a 16-byte multiple length.  So each stage row of each strip is ONE bulk copy of
// up to 400 bytes from the row's 16-byte aligned-down start, issued by its own lane
// (lane = strip * CH + row: the whole stage is one warp instruction), completing on the
// stage mbarrier as transaction bytes like a TMA box.  The consumer undoes the per-row
// skew (0..15 bytes, advancing by pitch mod 16 per row) with a word offset and a funnel
// shift, then runs the u8 core of the TMA path unchanged (G = 1: scalar, G = 2: packed
// dual-strip).  The view's end: bulk_stage_fill (STRICT).  Rows below the image are not
// copied and columns beyond the row end are stale — neither reaches a stored output.

template <bool EXACT, int CH, int G, bool STRICT = false>
struct U8BulkOp : std::conditional_t<G == 2, HarrisU8x2Op<EXACT, CH, 124>, HarrisU8Op<EXACT, CH, 124>> {
    using Base = std::conditional_t<G == 2, HarrisU8x2Op<EXACT, CH, 124>, HarrisU8Op<EXACT, CH, 124>>;
    static_assert(G * CH <= 32, "one lane per stage row");
    static constexpr bool kWarpLoad = true;
    static constexpr int kBarArrivals = kBulkBarArrivals;
    static constexpr bool kCacheProducer = true;
    static constexpr int kRowWords = 100;  // 400 B >= 15 skew bytes + 128 px * 3 B, 16-byte multiple
    static constexpr uint32_t kBoxBytes = uint32_t(CH) * kRowWords * 4u;
    static constexpr uint32_t kBoxStride = (kBoxBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kStageBytes = uint32_t(G) * kBoxStride;
    struct Params {
        float kappa;
        const uint8_t* rgb;
        int64_t in_pitch, in_image_stride;  // bytes
        int32_t W, H;                       // input pixels per row / rows per image
        const void* limit;                  // one past the view's last byte
    };
    uint32_t base_r, pitch_r, image_r;  // byte address residues mod 16
    uint32_t skew_a = 0, skew_b = 0;    // current row's skew of strips A and B

    __device__ __forceinline__ explicit U8BulkOp(const Params& p)
        : Base(typename Base::Params{p.kappa}),
          base_r(uint32_t(reinterpret_cast<uintptr_t>(p.rgb)) & 15u),
          pitch_r(uint32_t(p.in_pitch) & 15u),
          image_r(uint32_t(p.in_image_stride) & 15u) {}

    __device__ __forceinline__ void begin_tile(const int (&col0)[G], int row0, const int (&image)[G]) {
        const uint32_t r = base_r + uint32_t(row0) * pitch_r;
        skew_a = (r + uint32_t(image[0]) * image_r + uint32_t(col0[0]) * 3u) & 15u;
        if constexpr (G == 2) skew_b = (r + uint32_t(image[1]) * image_r + uint32_t(col0[1]) * 3u) & 15u;
    }

    __device__ __forceinline__ static void load_warp(void* smem, const Params& p, uint64_t* bar,
                                                     const int (&col0)[G], int row0, const int (&image)[G],
                                                     int lane, uint64_t policy) {
        const int k = lane >= CH ? 1 : 0, r = lane - k * CH;
        const int y = row0 + r;
        const int img = k ? image[G - 1] : image[0], c0 = k ? col0[G - 1] : col0[0];  // selects: no local array
        const uint8_t* src = p.rgb + int64_t(img) * p.in_image_stride + int64_t(y) * p.in_pitch + int64_t(c0) * 3;
        bulk_stage_fill<STRICT>(static_cast<unsigned char*>(smem) + k * kBoxStride + r * (kRowWords * 4), src,
                        uint32_t(p.W - c0) * 3u, kRowWords * 4, p.limit, bar, lane < G * CH && y < p.H,
                        row0 + CH > p.H - 1 && row0 <= p.H - 1, y == p.H - 1, lane);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[G][4]) {
        const uint32_t* wa = reinterpret_cast<const uint32_t*>(stage) + R * kRowWords + (skew_a >> 2) + 3 * lane;
        const uint32_t sa = (skew_a & 3u) * 8u;
        const uint32_t wa3 = wa[3];
        const uint32_t a[3] = {__funnelshift_r(wa[0], wa[1], sa), __funnelshift_r(wa[1], wa[2], sa),
                               __funnelshift_r(wa[2], wa3, sa)};
        skew_a = (skew_a + pitch_r) & 15u;
        if constexpr (G == 2) {
            const uint32_t* wb =
                reinterpret_cast<const uint32_t*>(stage + kBoxStride) + R * kRowWords + (skew_b >> 2) + 3 * lane;
            const uint32_t sb = (skew_b & 3u) * 8u;
            const uint32_t wb3 = wb[3];
            const uint32_t b[3] = {__funnelshift_r(wb[0], wb[1], sb), __funnelshift_r(wb[1], wb[2], sb),
                                   __funnelshift_r(wb[2], wb3, sb)};
            skew_b = (skew_b + pitch_r) & 15u;
            float2 gown[4];
            gray4_u8x2<EXACT>(a, b, gown[0], gown[1], gown[2], gown[3]);
            this->core.template step<R, NoHalo, (CH % 2 == 0)>(gown, lane, NoHalo{}, out);
        } else {
            float gown[4];
            gray4_u8<EXACT>(a[0], a[1], a[2], gown[0], gown[1], gown[2], gown[3]);
            this->core.template step<R, NoHalo, (CH % 2 == 0)>(gown, lane, NoHalo{}, out[0]);
        }
    }
};

#ifndef HARRIS_U8BULK_G
// scalar core, 16 warps/SM: 613 k vs 610 k (dual, 8 warps) on 512 x 1080x1918, 578 k vs 543 k
// on 8192x8191
#define HARRIS_U8BULK_G 1
#endif
constexpr int kU8BulkG = HARRIS_U8BULK_G;
constexpr int kU8BulkNW = 8, kU8BulkNS = 4, kU8BulkCH = 6, kU8BulkMinB = kU8BulkG == 2 ? 1 : 2;
const TmaConfig kU8BulkConfig = {kU8BulkNW, kU8BulkNS, kU8BulkCH, kU8BulkG, 124};
template <bool EXACT, bool STRICT = false>
using U8BulkOpT = U8BulkOp<EXACT, kU8BulkCH, kU8BulkG, STRICT>;

template <bool EXACT, bool STRICT = false>
static constexpr auto u8_bulk_kernel() {
    return strip_kernel<U8BulkOpT<EXACT, STRICT>, kU8BulkNW, kU8BulkNS, kU8BulkMinB>;
}
static constexpr size_t u8_bulk_smem() {
    return StripShape<kU8BulkNW, kU8BulkNS, U8BulkOpT<false>>::kSmemBytes;
}
static_assert(u8_bulk_smem() <= 227 * 1024, "u8 bulk smem");

constexpr int kU8LdgNW = 8, kU8LdgNS = 4, kU8LdgCH = 6;
const TmaConfig kU8LdgConfig = {kU8LdgNW, kU8LdgNS, kU8LdgCH, 1, 124};

template <bool EXACT, int A>
static constexpr auto u8_ldg_kernel() {
    return strip_kernel<U8LdgOp<EXACT, kU8LdgCH, A>, kU8LdgNW, kU8LdgNS, 2>;
}
static constexpr size_t u8_ldg_smem() {
    return StripShape<kU8LdgNW, kU8LdgNS, U8LdgOp<false, kU8LdgCH, 4>>::kSmemBytes;
}
static_assert(u8_ldg_smem() <= 227 * 1024, "u8 ldg smem");

template <int A>
static cudaError_t u8_ldg_configure_one() {
    cudaError_t e = cudaFuncSetAttribute(u8_ldg_kernel<false, A>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(u8_ldg_smem()));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(u8_ldg_kernel<true, A>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(u8_ldg_smem()));
    return e;
}

cudaError_t u8_ldg_configure(int* ctas_per_sm, int* bulk_ctas_per_sm) {
    cudaError_t e = u8_ldg_configure_one<4>();
    if (e == cudaSuccess) e = u8_ldg_configure_one<16>();
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, u8_ldg_kernel<false, 16>(), kU8LdgNW * 32,
                                                          u8_ldg_smem());
    for (const void* k : {reinterpret_cast<const void*>(u8_bulk_kernel<false, false>()), reinterpret_cast<const void*>(u8_bulk_kernel<true, false>()), reinterpret_cast<const void*>(u8_bulk_kernel<false, true>()), reinterpret_cast<const void*>(u8_bulk_kernel<true, true>())})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(u8_bulk_smem()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(bulk_ctas_per_sm, u8_bulk_kernel<false>(), kU8BulkNW * 32,
                                                          u8_bulk_smem());
    return e;
}

template <bool EXACT, int A>
static void launch_u8_ldg_one(const Geom& geom, const TileGeom& tg, int64_t grid, cudaStream_t stream) {
    CUtensorMap unused;
    std::memset(&unused, 0, sizeof(unused));
    const int64_t img_stride = geom.batch > 1 ? geom.in_image_stride : 0;
    const typename U8LdgOp<EXACT, kU8LdgCH, A>::Params p{geom.kappa, reinterpret_cast<const uint8_t*>(geom.rgb),
                                                         geom.in_pitch, img_stride, int32_t(geom.m + 4),
                                                         int32_t(geom.n + 4)};
    launch_strip(u8_ldg_kernel<EXACT, A>(), unsigned(grid), unsigned(kU8LdgNW * 32), u8_ldg_smem(), stream, tg.pdl, unused, tg, p);
}

template <bool EXACT>
static void launch_u8_bulk_one(const Geom& geom, const TileGeom& tg, int64_t grid, cudaStream_t stream) {
    CUtensorMap unused;
    std::memset(&unused, 0, sizeof(unused));
    const int64_t img_stride = geom.batch > 1 ? geom.in_image_stride : 0;
    const uint8_t* rgb = reinterpret_cast<const uint8_t*>(geom.rgb);
    const uint8_t* limit = rgb + (geom.batch - 1) * img_stride + (geom.n + 3) * geom.in_pitch + 3 * (geom.m + 4);
    auto go = [&](auto strict) {
        constexpr bool S = decltype(strict)::value;
        const typename U8BulkOpT<EXACT, S>::Params p{geom.kappa, rgb, geom.in_pitch, img_stride, int32_t(geom.m + 4),
                                                     int32_t(geom.n + 4), limit};
        launch_strip(u8_bulk_kernel<EXACT, S>(), unsigned(grid), unsigned(kU8BulkNW * 32), u8_bulk_smem(), stream, tg.pdl, unused, tg, p);
    };
    // STRICT only when the 16-byte rounding could pass the view's end
    (reinterpret_cast<uintptr_t>(limit) & 15u) ? go(std::true_type{}) : go(std::false_type{});
}

// chunk 0: the bulk-copy kernel (K1b, default); 4 / 16: the cp.async kernel (K2)
cudaError_t launch_u8_ldg(bool exact, int chunk, const Geom& geom, const TileGeom& tg, int64_t grid,
                          cudaStream_t stream) {
    if (chunk == 0)
        exact ? launch_u8_bulk_one<true>(geom, tg, grid, stream) : launch_u8_bulk_one<false>(geom, tg, grid, stream);
    else if (chunk == 4)
        exact ? launch_u8_ldg_one<true, 4>(geom, tg, grid, stream) : launch_u8_ldg_one<false, 4>(geom, tg, grid, stream);
    else
        exact ? launch_u8_ldg_one<true, 16>(geom, tg, grid, stream)
              : launch_u8_ldg_one<false, 16>(geom, tg, grid, stream);
    return cudaGetLastError();
}

// configs: 0 = packed dual-strip core (8 warps/SM), 1 = scalar core (2 x 8 warps/SM)
template <int CFG>
struct LdgCfg;
template <>
struct LdgCfg<0> {
    static constexpr int NW = 8, NS = 2, CH = 3, MINB = 1, G = 2;
    template <bool EXACT, bool STRICT = false>
    using Op = LdgOp<HarrisF32x2Op<EXACT, CH, 128>, 4>;
};
template <>
struct LdgCfg<1> {
    static constexpr int NW = 8, NS = 2, CH = 3, MINB = 2, G = 1;
    template <bool EXACT, bool STRICT = false>
    using Op = LdgOp<HarrisF32Op<EXACT, CH, 128>, 4>;
};

// 2 = scalar core in the 124-column lane-halo layout: 128-column rows are exactly 4
// copies per lane (132 need a 5th), and the halo branch disappears
template <>
struct LdgCfg<2> {
    static constexpr int NW = 8, NS = 2, CH = 3, MINB = 2, G = 1;
    template <bool EXACT, bool STRICT = false>
    using Op = LdgOp<HarrisF32Op<EXACT, CH, 124>, 4>;
};

// 3 / 4 = the bulk-copy engine (K1b) with the scalar / packed dual-strip core
template <>
struct LdgCfg<3> {
    static constexpr int NW = 8, NS = 2, CH = 3, MINB = 2, G = 1;
    template <bool EXACT, bool STRICT = false>
    using Op = F32BulkOp<EXACT, CH, 1, STRICT>;
};
template <>
struct LdgCfg<4> {
    static constexpr int NW = 8, NS = 2, CH = 3, MINB = 1, G = 2;
    template <bool EXACT, bool STRICT = false>
    using Op = F32BulkOp<EXACT, CH, 2, STRICT>;
};

const TmaConfig kLdgConfigs[kNumLdgConfigs] = {
    {8, 2, 3, 2, 128}, {8, 2, 3, 1, 128}, {8, 2, 3, 1, 124}, {8, 2, 3, 1, 124}, {8, 2, 3, 2, 124}};

template <int CFG, bool EXACT, bool STRICT = false>
static constexpr auto ldg_kernel() {
    using C = LdgCfg<CFG>;
    return strip_kernel<typename C::template Op<EXACT, STRICT>, C::NW, C::NS, C::MINB>;
}
template <int CFG>
static constexpr size_t ldg_smem() {
    using C = LdgCfg<CFG>;
    return StripShape<C::NW, C::NS, typename C::template Op<false>>::kSmemBytes;
}
static_assert(ldg_smem<0>() <= 227 * 1024 && ldg_smem<1>() <= 227 * 1024 && ldg_smem<2>() <= 227 * 1024 &&
                  ldg_smem<3>() <= 227 * 1024 && ldg_smem<4>() <= 227 * 1024,
              "ldg smem");

template <int CFG>
static cudaError_t ldg_configure_one(int* ctas_per_sm) {
    cudaError_t e = cudaSuccess;
    for (const void* k : {reinterpret_cast<const void*>(ldg_kernel<CFG, false, false>()), reinterpret_cast<const void*>(ldg_kernel<CFG, true, false>()), reinterpret_cast<const void*>(ldg_kernel<CFG, false, true>()), reinterpret_cast<const void*>(ldg_kernel<CFG, true, true>())})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ldg_smem<CFG>()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, ldg_kernel<CFG, false>(), LdgCfg<CFG>::NW * 32,
                                                          ldg_smem<CFG>());
    return e;
}

cudaError_t ldg_configure(int cfg, int* ctas_per_sm) {
    return cfg == 0   ? ldg_configure_one<0>(ctas_per_sm)
           : cfg == 1 ? ldg_configure_one<1>(ctas_per_sm)
           : cfg == 2 ? ldg_configure_one<2>(ctas_per_sm)
           : cfg == 3 ? ldg_configure_one<3>(ctas_per_sm)
                      : ldg_configure_one<4>(ctas_per_sm);
}

template <int CFG, bool EXACT>
static void launch_ldg_one(const Geom& geom, const TileGeom& tg, int64_t grid, cudaStream_t stream) {
    CUtensorMap unused;
    std::memset(&unused, 0, sizeof(unused));
    const int64_t img_stride = geom.batch > 1 ? geom.in_image_stride : 0;
    const float* limit = geom.rgb + (geom.batch - 1) * img_stride + 2 * geom.in_chan_stride +
                         (geom.n + 3) * geom.in_pitch + (geom.m + 4);
    auto go = [&](auto strict) {
        constexpr bool S = decltype(strict)::value;
        using Op = typename LdgCfg<CFG>::template Op<EXACT, S>;
        const typename Op::Params p{{geom.kappa}, geom.rgb, geom.in_pitch, geom.in_chan_stride, img_stride,
                                    int32_t(geom.m + 4), int32_t(geom.n + 4), limit};
        launch_strip(ldg_kernel<CFG, EXACT, S>(), unsigned(grid), unsigned(LdgCfg<CFG>::NW * 32), ldg_smem<CFG>(), stream, tg.pdl, unused, tg, p);
    };
    (reinterpret_cast<uintptr_t>(limit) & 15u) ? go(std::true_type{}) : go(std::false_type{});
}

cudaError_t launch_ldg(int cfg, bool exact, const Geom& geom, const TileGeom& tg, int64_t grid,
                       cudaStream_t stream) {
    if (cfg == 0)
        exact ? launch_ldg_one<0, true>(geom, tg, grid, stream) : launch_ldg_one<0, false>(geom, tg, grid, stream);
    else if (cfg == 1)
        exact ? launch_ldg_one<1, true>(geom, tg, grid, stream) : launch_ldg_one<1, false>(geom, tg, grid, stream);
    else if (cfg == 2)
        exact ? launch_ldg_one<2, true>(geom, tg, grid, stream) : launch_ldg_one<2, false>(geom, tg, grid, stream);
    else if (cfg == 3)
        exact ? launch_ldg_one<3, true>(geom, tg, grid, stream) : launch_ldg_one<3, false>(geom, tg, grid, stream);
    else
        exact ? launch_ldg_one<4, true>(geom, tg, grid, stream) : launch_ldg_one<4, false>(geom, tg, grid, stream);
    return cudaGetLastError();
}

// ---- separable 3x3 stencil through the bulk-copy engine (K1b): one cp.async.bulk per
// stage row (<= 544 B from the 16-byte aligned-down start), the consumer reads its 6
// floats at the row's float skew (even: three 8-byte loads; odd: scalar + 2 x 8-byte +
// scalar) and runs the unchanged Sep3x3Op arithmetic
template <bool EXACT, int CH, bool STRICT = false>
struct SepBulkOp : Sep3x3Op<EXACT, CH> {
    using Base = Sep3x3Op<EXACT, CH>;
    static_assert(CH <= 32, "one lane per stage row");
    static constexpr bool kWarpLoad = true;
    static constexpr int kBarArrivals = kBulkBarArrivals;
    static constexpr bool kCacheProducer = true;
    static constexpr int kRowFloats = 136;  // 3 skew floats + 130 columns, 16-byte multiple
    static constexpr uint32_t kStageBytes = (uint32_t(CH) * kRowFloats * 4u + 127u) / 128u * 128u;
    struct Params {
        typename Base::Params base;
        const float* src;
        int64_t in_pitch, in_plane_stride, in_image_stride;  // elements (plane stride unused)
        int32_t W, H;
        const void* limit;  // one past the view's last element
    };
    uint32_t base_r, pitch_r, image_r, sk = 0;

    __device__ __forceinline__ explicit SepBulkOp(const Params& p)
        : Base(p.base),
          base_r(uint32_t(reinterpret_cast<uintptr_t>(p.src) >> 2) & 3u),
          pitch_r(uint32_t(p.in_pitch) & 3u),
          image_r(uint32_t(p.in_image_stride) & 3u) {}

    __device__ __forceinline__ void begin_tile(const int (&col0)[1], int row0, const int (&image)[1]) {
        sk = (base_r + uint32_t(image[0]) * image_r + uint32_t(row0) * pitch_r + uint32_t(col0[0])) & 3u;
    }

    __device__ __forceinline__ static void load_warp(void* smem, const Params& p, uint64_t* bar,
                                                     const int (&col0)[1], int row0, const int (&image)[1],
                                                     int lane, uint64_t policy) {
        const int y = row0 + lane;
        const float* src = p.src + int64_t(image[0]) * p.in_image_stride + int64_t(y) * p.in_pitch + col0[0];
        bulk_stage_fill<STRICT>(static_cast<unsigned char*>(smem) + lane * (kRowFloats * 4), src, uint32_t(p.W - col0[0]) * 4u,
                        kRowFloats * 4, p.limit, bar, lane < CH && y < p.H,
                        row0 + CH > p.H - 1 && row0 <= p.H - 1, y == p.H - 1, lane);
    }

    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out4)[1][4]) {
        const float* q = reinterpret_cast<const float*>(stage) + R * kRowFloats + 4 * lane;
        float x[6];
        if (sk & 1u) {
            const float2 u = lds64(q + sk + 1), v = lds64(q + sk + 3);
            x[0] = q[sk], x[1] = u.x, x[2] = u.y, x[3] = v.x, x[4] = v.y, x[5] = q[sk + 5];
        } else {
            const float2 u = lds64(q + sk), v = lds64(q + sk + 2), w = lds64(q + sk + 4);
            x[0] = u.x, x[1] = u.y, x[2] = v.x, x[3] = v.y, x[4] = w.x, x[5] = w.y;
        }
        sk = (sk + pitch_r) & 3u;
        this->template compute<R>(x, out4[0]);
    }
};

// ---- separable 3x3 stencil on planes TMA cannot describe (pitch % 4 != 0 / base) ----
constexpr int kSepLdgNW = 8, kSepLdgNS = 8, kSepLdgCH = 6;
const TmaConfig kSepLdgConfig = {kSepLdgNW, kSepLdgNS, kSepLdgCH, 1, 128};

template <bool EXACT, bool STRICT = false>
using SepLdgOpT = SepBulkOp<EXACT, kSepLdgCH, STRICT>;

template <bool EXACT, bool STRICT = false>
static constexpr auto sep_ldg_kernel() {
    return strip_kernel<SepLdgOpT<EXACT, STRICT>, kSepLdgNW, kSepLdgNS, 1>;
}
static constexpr size_t sep_ldg_smem() {
    return StripShape<kSepLdgNW, kSepLdgNS, SepLdgOpT<false>>::kSmemBytes;
}
static_assert(sep_ldg_smem() <= 227 * 1024, "stencil ldg smem");

cudaError_t sep_ldg_configure(int* ctas_per_sm) {
    cudaError_t e = cudaSuccess;
    for (const void* k : {reinterpret_cast<const void*>(sep_ldg_kernel<false, false>()), reinterpret_cast<const void*>(sep_ldg_kernel<true, false>()), reinterpret_cast<const void*>(sep_ldg_kernel<false, true>()), reinterpret_cast<const void*>(sep_ldg_kernel<true, true>())})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sep_ldg_smem()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, sep_ldg_kernel<false>(), kSepLdgNW * 32,
                                                          sep_ldg_smem());
    return e;
}

template <bool EXACT>
static void launch_sep_ldg_one(const float* in, int64_t in_pitch, int64_t in_image_stride, int32_t W, int32_t H,
                               const TileGeom& tg, int64_t grid, const float* wv, const float* wh,
                               cudaStream_t stream) {
    CUtensorMap unused;
    std::memset(&unused, 0, sizeof(unused));
    const int64_t img_stride = tg.batch > 1 ? in_image_stride : 0;
    const float* limit = in + (tg.batch - 1) * img_stride + int64_t(H - 1) * in_pitch + W;
    auto go = [&](auto strict) {
        constexpr bool S = decltype(strict)::value;
        using Op = SepLdgOpT<EXACT, S>;
        const typename Op::Params p{{{wv[0], wv[1], wv[2]}, {wh[0], wh[1], wh[2]}}, in, in_pitch, 0, img_stride, W,
                                    H, limit};
        launch_strip(sep_ldg_kernel<EXACT, S>(), unsigned(grid), unsigned(kSepLdgNW * 32), sep_ldg_smem(), stream, tg.pdl, unused, tg, p);
    };
    (reinterpret_cast<uintptr_t>(limit) & 15u) ? go(std::true_type{}) : go(std::false_type{});
}

cudaError_t launch_sep_ldg(bool exact, const float* in, int64_t in_pitch, int64_t in_image_stride, int64_t W,
                           int64_t H, const TileGeom& tg, int64_t grid, const float* wv, const float* wh,
                           cudaStream_t stream) {
    if (exact)
        launch_sep_ldg_one<true>(in, in_pitch, in_image_stride, int32_t(W), int32_t(H), tg, grid, wv, wh, stream);
    else
        launch_sep_ldg_one<false>(in, in_pitch, in_image_stride, int32_t(W), int32_t(H), tg, grid, wv, wh, stream);
    return cudaGetLastError();
}

}  // namespace harris
