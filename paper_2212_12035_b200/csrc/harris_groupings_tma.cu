// harris_groupings_tma.cu — the thesis's kernel groupings built from
// bandwidth-optimised kernels, for a FAIR fusion ablation.
//
// harris_groupings.cu holds one deliberately simple kernel per group (one thread per pixel,
// Appendix-B order): a fused-vs-naive comparison.  Here every group is a strip-engine op
// (strip_pipeline.cuh: per-warp TMA ring, register row rotation, 16-byte stores) in the FAST
// arithmetic of the fused kernel, so the ablation measures fusion alone:
//
//   1  [Sx] [Sy] [x] [+] [coarsity]   SobelGroupOp<kIx>, SobelGroupOp<kIy>, ProdGroupOp,
//                                     BoxGroupOp<false>, CoarsGroupOp
//   2  [Sx,Sy,x] [+,coarsity]         SobelGroupOp<kProd>, BoxGroupOp<true>
//   3  [Sx,Sy] [x,+,coarsity]         SobelGroupOp<kIxIy>, PbcGroupOp
//   4  fused                          harris_run (the product kernel)
//
// Arithmetic: Ix / Iy are bit-identical to the fused kernel's (same gray, same separable
// Sobel); grouping 3's second kernel is the fused core's back half (products folded into the
// shared-pair horizontal sums), so grouping 3 equals the fused FAST output bit for bit;
// groupings 1 and 2 materialise rounded products (and box sums), which the fused kernel never
// rounds, so they agree with it within the SURVEY.md §8(d) tolerance.
//
// Intermediates live in caller scratch as planes with a 16-byte aligned pitch (the TMA
// tensor maps of the next group need it): Ix, Iy and the products are (n+2) x pitch_s planes,
// the box sums n x pitch_o; grouping_fast_scratch_floats() gives the sizes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "harris_common.cuh"
#include "harris_internal.h"
#include "harris_ops.cuh"
#include "strip_pipeline.cuh"

namespace harris {

namespace {

constexpr int kGrpCH = 3, kGrpNW = 8, kGrpNS = 4;

// the common TMA stage of every group op: one 4-D box {BOX cols, CH rows, PIN planes, 1}
template <int PIN, int BOX, int CH>
struct GroupStage {
    static_assert(CH % 3 == 0, "row rotation needs CH % 3 == 0");
    static constexpr int kGroups = 1;
    static constexpr int kStripCols = kWarpCols;
    static constexpr int kRowsPerStage = CH;
    static constexpr int kBox = BOX;
    static constexpr uint32_t kTxBytes = uint32_t(PIN) * CH * BOX * 4u;
    static constexpr uint32_t kStageBytes = (kTxBytes + 127u) / 128u * 128u;
    struct Params {
        float kappa;
    };
    __device__ __forceinline__ static void load(void* smem, const CUtensorMap* tmap, uint64_t* bar,
                                                const int (&col0)[1], int row0, const int (&image)[1],
                                                uint64_t policy) {
        tma_load_4d(smem, tmap, bar, col0[0], row0, 0, image[0], policy);
    }
    // plane p, row R of the stage, this lane's 4 columns (+ the next 2 from lane + 1; lane 31
    // reads box columns 128, 129 — only for BOX == 132)
    template <int R>
    __device__ __forceinline__ static void row6(const unsigned char* stage, int p, int lane, float (&v)[6]) {
        const float* q = reinterpret_cast<const float*>(stage) + (p * CH + R) * BOX;
        const float4 a = lds128(q + lane * 4);
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
        v[4] = __shfl_down_sync(0xffffffffu, v[0], 1);
        v[5] = __shfl_down_sync(0xffffffffu, v[1], 1);
        if constexpr (BOX > kWarpCols) {
            if (lane == 31) {
                const float2 h = lds64(q + kWarpCols);
                v[4] = h.x, v[5] = h.y;
            }
        }
    }
    template <int R>
    __device__ __forceinline__ static float4 row4(const unsigned char* stage, int p, int lane) {
        return lds128(reinterpret_cast<const float*>(stage) + (p * CH + R) * BOX + lane * 4);
    }
};

enum SobelMode { kIx = 1, kIy = 2, kIxIy = 3, kProd = 4 };

// [Sx] / [Sy] / [Sx,Sy] / [Sx,Sy,x]: planar RGB -> Ix and/or Iy or the three products.
// Gray and the separable Sobel in the fused kernel's FAST arithmetic (HarrisCore).
template <int MODE>
struct SobelGroupOp : GroupStage<3, kBoxCols, kGrpCH> {
    using S = GroupStage<3, kBoxCols, kGrpCH>;
    static constexpr int kHaloRows = 2;
    static constexpr int kOutPlanes = MODE == kIxIy ? 2 : MODE == kProd ? 3 : 1;
    float D[3][4], Hs[3][4];
    __device__ __forceinline__ explicit SobelGroupOp(const typename S::Params&) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 4; ++k) D[a][k] = Hs[a][k] = 0.f;
    }
    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[kOutPlanes][4]) {
        constexpr int s2 = R % 3, s0 = (R + 1) % 3, s1 = (R + 2) % 3;
        float r[6], g[6], b[6], gr[6];
        S::template row6<R>(stage, 0, lane, r);
        S::template row6<R>(stage, 1, lane, g);
        S::template row6<R>(stage, 2, lane, b);
#pragma unroll
        for (int k = 0; k < 6; ++k) gr[k] = gray_of<false>(r[k], g[k], b[k]);
        float ix[4], iy[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            D[s2][k] = gr[k + 2] - gr[k];
            Hs[s2][k] = fmaf(2.f, gr[k + 1], gr[k]) + gr[k + 2];
            ix[k] = fmaf(2.f, D[s1][k], D[s0][k] + D[s2][k]);
            iy[k] = Hs[s2][k] - Hs[s0][k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if constexpr (MODE == kIx) {
                out[0][k] = ix[k];
            } else if constexpr (MODE == kIy) {
                out[0][k] = iy[k];
            } else if constexpr (MODE == kIxIy) {
                out[0][k] = ix[k];
                out[1][k] = iy[k];
            } else {
                out[0][k] = ix[k] * ix[k];
                out[1][k] = ix[k] * iy[k];
                out[2][k] = iy[k] * iy[k];
            }
        }
    }
};

// [x]: Ix, Iy -> the three products (pointwise)
struct ProdGroupOp : GroupStage<2, kWarpCols, kGrpCH> {
    using S = GroupStage<2, kWarpCols, kGrpCH>;
    static constexpr int kHaloRows = 0;
    static constexpr int kOutPlanes = 3;
    __device__ __forceinline__ explicit ProdGroupOp(const typename S::Params&) {}
    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[3][4]) {
        const float4 a = S::template row4<R>(stage, 0, lane), b = S::template row4<R>(stage, 1, lane);
        const float x[4] = {a.x, a.y, a.z, a.w}, y[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            out[0][k] = x[k] * x[k];
            out[1][k] = x[k] * y[k];
            out[2][k] = y[k] * y[k];
        }
    }
};

// [+] / [+,coarsity]: the three product planes -> the box sums (3 planes) or the coarsity;
// FAST box sums as in the fused core (shared-pair horizontal 3-sums, then vertical)
template <bool COARS>
struct BoxGroupOp : GroupStage<3, kBoxCols, kGrpCH> {
    using S = GroupStage<3, kBoxCols, kGrpCH>;
    static constexpr int kHaloRows = 2;
    static constexpr int kOutPlanes = COARS ? 1 : 3;
    float kappa;
    float HB[3][12];
    __device__ __forceinline__ explicit BoxGroupOp(const typename S::Params& p) : kappa(p.kappa) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 12; ++k) HB[a][k] = 0.f;
    }
    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[kOutPlanes][4]) {
        constexpr int s2 = R % 3, s0 = (R + 1) % 3, s1 = (R + 2) % 3;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            float v[6];
            S::template row6<R>(stage, q, lane, v);
            hsum4(v, HB[s2][4 * q + 0], HB[s2][4 * q + 1], HB[s2][4 * q + 2], HB[s2][4 * q + 3]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float sxx = (HB[s0][0 + j] + HB[s1][0 + j]) + HB[s2][0 + j];
            const float sxy = (HB[s0][4 + j] + HB[s1][4 + j]) + HB[s2][4 + j];
            const float syy = (HB[s0][8 + j] + HB[s1][8 + j]) + HB[s2][8 + j];
            if constexpr (COARS) {
                out[0][j] = coarsity_fast(sxx, sxy, syy, kappa);
            } else {
                out[0][j] = sxx;
                out[1][j] = sxy;
                out[2][j] = syy;
            }
        }
    }
};

// [coarsity]: the three box-sum planes -> coarsity (pointwise)
struct CoarsGroupOp : GroupStage<3, kWarpCols, kGrpCH> {
    using S = GroupStage<3, kWarpCols, kGrpCH>;
    static constexpr int kHaloRows = 0;
    float kappa;
    __device__ __forceinline__ explicit CoarsGroupOp(const typename S::Params& p) : kappa(p.kappa) {}
    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        const float4 a = S::template row4<R>(stage, 0, lane), b = S::template row4<R>(stage, 1, lane),
                     c = S::template row4<R>(stage, 2, lane);
        out[0][0] = coarsity_fast(a.x, b.x, c.x, kappa);
        out[0][1] = coarsity_fast(a.y, b.y, c.y, kappa);
        out[0][2] = coarsity_fast(a.z, b.z, c.z, kappa);
        out[0][3] = coarsity_fast(a.w, b.w, c.w, kappa);
    }
};

// [x,+,coarsity]: Ix, Iy -> coarsity, the fused core's back half (products folded into the
// shared-pair horizontal sums, vertical sums, coarsity): bit-identical to the fused FAST output
struct PbcGroupOp : GroupStage<2, kBoxCols, kGrpCH> {
    using S = GroupStage<2, kBoxCols, kGrpCH>;
    static constexpr int kHaloRows = 2;
    float kappa;
    float HB[3][12];
    __device__ __forceinline__ explicit PbcGroupOp(const typename S::Params& p) : kappa(p.kappa) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 12; ++k) HB[a][k] = 0.f;
    }
    template <int R>
    __device__ __forceinline__ void row(const unsigned char* stage, int lane, float (&out)[1][4]) {
        constexpr int s2 = R % 3, s0 = (R + 1) % 3, s1 = (R + 2) % 3;
        float ix[6], iy[6];
        S::template row6<R>(stage, 0, lane, ix);
        S::template row6<R>(stage, 1, lane, iy);
        prodsum4(ix, ix, HB[s2][0], HB[s2][1], HB[s2][2], HB[s2][3]);
        prodsum4(ix, iy, HB[s2][4], HB[s2][5], HB[s2][6], HB[s2][7]);
        prodsum4(iy, iy, HB[s2][8], HB[s2][9], HB[s2][10], HB[s2][11]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float sxx = (HB[s0][0 + j] + HB[s1][0 + j]) + HB[s2][0 + j];
            const float sxy = (HB[s0][4 + j] + HB[s1][4 + j]) + HB[s2][4 + j];
            const float syy = (HB[s0][8 + j] + HB[s1][8 + j]) + HB[s2][8 + j];
            out[0][j] = coarsity_fast(sxx, sxy, syy, kappa);
        }
    }
};

template <class T>
struct OpTag {
    using type = T;
};

template <class Op>
constexpr auto grp_kernel() {
    return strip_kernel<Op, kGrpNW, kGrpNS, 1>;
}
template <class Op>
constexpr size_t grp_smem() {
    return StripShape<kGrpNW, kGrpNS, Op>::kSmemBytes;
}

template <class Op>
cudaError_t grp_configure_one(int* occ) {
    cudaError_t e = cudaFuncSetAttribute(grp_kernel<Op>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(grp_smem<Op>()));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, grp_kernel<Op>(), kGrpNW * 32, grp_smem<Op>());
    return e;
}

// scratch plane geometry (elements): 16-byte aligned pitches, 256-byte aligned planes
struct GrpLayout {
    int64_t Hs, Ws, ps, ss;  // Sobel-sized planes: rows, cols, pitch, plane stride
    int64_t n, m, po, so;    // output-sized planes
    GrpLayout(int64_t n_, int64_t m_) : n(n_), m(m_) {
        Hs = n + 2;
        Ws = m + 2;
        ps = (Ws + 3) / 4 * 4;
        ss = (ps * Hs + 63) / 64 * 64;
        po = (m + 3) / 4 * 4;
        so = (po * n + 63) / 64 * 64;
    }
};

}  // namespace

int64_t grouping_fast_scratch_floats(int grouping, int64_t n, int64_t m) {
    const GrpLayout L(n, m);
    switch (grouping) {
        case 1: return 2 * L.ss + 3 * L.ss + 3 * L.so;  // Ix, Iy, products, box sums
        case 2: return 3 * L.ss;                        // products
        case 3: return 2 * L.ss;                        // Ix, Iy
        case 4: return 0;
        default: return -1;
    }
}

cudaError_t grouping_fast_configure(int* occ) {
    // all group ops share the pipeline shape; the 3-plane, 132-column stage is the largest
    int o = 0;
    cudaError_t e = grp_configure_one<SobelGroupOp<kIx>>(&o);
    if (e == cudaSuccess) e = grp_configure_one<SobelGroupOp<kIy>>(&o);
    if (e == cudaSuccess) e = grp_configure_one<SobelGroupOp<kIxIy>>(&o);
    if (e == cudaSuccess) e = grp_configure_one<SobelGroupOp<kProd>>(&o);
    if (e == cudaSuccess) e = grp_configure_one<ProdGroupOp>(&o);
    if (e == cudaSuccess) e = grp_configure_one<BoxGroupOp<false>>(&o);
    if (e == cudaSuccess) e = grp_configure_one<BoxGroupOp<true>>(&o);
    if (e == cudaSuccess) e = grp_configure_one<CoarsGroupOp>(&o);
    if (e == cudaSuccess) e = grp_configure_one<PbcGroupOp>(&o);
    if (e == cudaSuccess) e = grp_configure_one<SobelGroupOp<kProd>>(occ);  // the lowest occupancy
    return e;
}

// one group launch: tensor map over `planes` planes of `rows` x `cols` at `src` (pitch, plane
// stride in elements), output rows x cols planes at `dst`
template <class Op>
static int grp_launch(const GroupLaunchEnv& env, const float* src, int64_t in_rows, int64_t in_cols,
                      int64_t in_pitch, int64_t in_plane_stride, int planes, float* dst, int64_t out_rows,
                      int64_t out_cols, int64_t out_pitch, int64_t out_plane_stride, float kappa,
                      cudaStream_t stream) {
    CUtensorMap tmap;
    cuuint64_t dims[4] = {cuuint64_t(in_cols), cuuint64_t(in_rows), cuuint64_t(planes), 1};
    cuuint64_t strides[3] = {cuuint64_t(in_pitch) * 4, cuuint64_t(in_plane_stride) * 4,
                             cuuint64_t(in_plane_stride) * planes * 4};
    cuuint32_t box[4] = {cuuint32_t(Op::kBox), cuuint32_t(kGrpCH), cuuint32_t(planes), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = env.encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(src), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -1;
    TileGeom tg;
    const int64_t resident = int64_t(env.num_sms) * (env.occ > 0 ? env.occ : 1);
    plan_tiles_ext(out_rows, out_cols, 1, resident * kGrpNW, kGrpCH, 0, tg, Op::kHaloRows);
    const int64_t grid = std::min<int64_t>((tg.tiles + kGrpNW - 1) / kGrpNW, resident);
    tg.out = dst;
    tg.out_pitch = out_pitch;
    tg.out_image_stride = out_rows * out_pitch;
    tg.out_plane_stride = out_plane_stride;
    tg.kappa = kappa;
    tg.l2_policy = env.l2_policy;
    tg.vec_store = store_mode_ext(dst, out_pitch, 1, 0);
    tg.sync_waves = 1;
    const typename Op::Params p{kappa};
    const cudaError_t e = launch_strip(grp_kernel<Op>(), dim3(unsigned(grid)), dim3(kGrpNW * 32), grp_smem<Op>(),
                                       stream, 0, tmap, tg, p);
    return e == cudaSuccess ? 0 : 1;
}

// FAST groupings 1-3 on one contiguous image (rgb 3 x (n+4) x (m+4), W % 4 == 0); returns 0,
// -1 (tensor-map encode failed) or 1 (launch failed, see cudaGetLastError)
int launch_grouping_fast(const GroupLaunchEnv& env, int grouping, float* out, int64_t n, int64_t m,
                         const float* rgb, float* scratch, float kappa, cudaStream_t st) {
    const GrpLayout L(n, m);
    const int64_t H = n + 4, W = m + 4;
    float* ixy = scratch;  // Ix at 0, Iy at ss
    int rc = 0;
    auto sobel = [&](auto tag, float* dst, int64_t plane_stride) {
        using Op = typename decltype(tag)::type;
        return grp_launch<Op>(env, rgb, H, W, W, H * W, 3, dst, L.Hs, L.Ws, L.ps, plane_stride, kappa, st);
    };
    switch (grouping) {
        case 1: {
            float* prod = ixy + 2 * L.ss;
            float* sums = prod + 3 * L.ss;
            rc = sobel(OpTag<SobelGroupOp<kIx>>{}, ixy, 0);
            if (!rc) rc = sobel(OpTag<SobelGroupOp<kIy>>{}, ixy + L.ss, 0);
            if (!rc)
                rc = grp_launch<ProdGroupOp>(env, ixy, L.Hs, L.Ws, L.ps, L.ss, 2, prod, L.Hs, L.Ws, L.ps, L.ss, kappa,
                                             st);
            if (!rc)
                rc = grp_launch<BoxGroupOp<false>>(env, prod, L.Hs, L.Ws, L.ps, L.ss, 3, sums, n, m, L.po, L.so, kappa,
                                                   st);
            if (!rc) rc = grp_launch<CoarsGroupOp>(env, sums, n, m, L.po, L.so, 3, out, n, m, m, 0, kappa, st);
            break;
        }
        case 2: {
            float* prod = scratch;
            rc = sobel(OpTag<SobelGroupOp<kProd>>{}, prod, L.ss);
            if (!rc)
                rc = grp_launch<BoxGroupOp<true>>(env, prod, L.Hs, L.Ws, L.ps, L.ss, 3, out, n, m, m, 0, kappa, st);
            break;
        }
        case 3:
            rc = sobel(OpTag<SobelGroupOp<kIxIy>>{}, ixy, L.ss);
            if (!rc) rc = grp_launch<PbcGroupOp>(env, ixy, L.Hs, L.Ws, L.ps, L.ss, 2, out, n, m, m, 0, kappa, st);
            break;
        default:
            return 2;
    }
    return rc;
}

}  // namespace harris
