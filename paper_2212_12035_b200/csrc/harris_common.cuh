// harris_common.cuh — arithmetic contract and sm_100a PTX helpers shared by the
// fused Harris kernels.
//
// Arithmetic (thesis PAPER.md:2346-2374 / 4587-4730):
//   g    = ((0.299f*R) + (0.587f*G)) + (0.114f*B)
//   Ix   = 9-tap SX accumulation from 0 in row-major order, SX = [[-a,0,a],[-b,0,b],[-a,0,a]]
//   Iy   = 9-tap SY = SX^T,  a = 0.083333336f (1/12), b = 0.16666667f (2/12)
//   S**  = 9-tap box sums of the products Ix*Ix, Ix*Iy, Iy*Iy, row-major from 0
//   out  = (Sxx*Syy - Sxy*Sxy) - (k*(Sxx+Syy))*(Sxx+Syy)
// EXACT mode evaluates exactly that with __fmul_rn/__fadd_rn (never contracted),
// so it is bit-identical to oracle/harris_oracle.c (-ffp-contract=off).  FAST
// mode uses the separable (cbuf+rrot) order with FMAs and the
// 1/12 Sobel scale folded into the gray weights; it is checked against the f64
// oracle under the SURVEY.md §8(d) tolerance.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace harris {

// thesis constants
constexpr float kGrayR = 0.299f, kGrayG = 0.587f, kGrayB = 0.114f;
constexpr float kSobA = 0.083333336f, kSobB = 0.16666667f;
// FAST mode: gray pre-scaled by 1/12 so the separable Sobel needs no final scale
constexpr float kGrayR12 = 0.299f / 12.0f, kGrayG12 = 0.587f / 12.0f, kGrayB12 = 0.114f / 12.0f;

constexpr int kLanes = 32;
constexpr int kColsPerLane = 4;                     // one float4 per lane
constexpr int kWarpCols = kLanes * kColsPerLane;    // 128 output columns per warp strip
constexpr int kBoxCols = kWarpCols + 4;             // + 4-column halo = 132 input columns
constexpr int kU8BoxWords = 100;  // u8 HWC box: 400 bytes >= 132 px * 3 B (TMA inner box: 16-B multiple)

// Strip layouts of the Harris ops (template parameter SC = output columns per strip):
//   SC = 128: every lane owns 4 output columns; lane 31 loads and converts the box's
//             4-column right halo itself (a divergent branch every row).
//   SC = 124: lane 31 owns the halo columns: it converts them like any other lane and
//             hands them to lane 30 through the same shuffle every lane uses, and stores
//             nothing.  No branch, no extra loads / gray math, 1/32 of the lanes idle.
// Box width = SC + 4 columns (f32: 132 / 128; u8: 100 / 96 words).
template <int SC>
struct Strip {
    static_assert(SC == 128 || SC == 124, "strip layouts: 128 or 124 columns");
    static constexpr int kCols = SC;
    static constexpr int kBoxCols = SC + 4;
    static constexpr bool kLaneHalo = SC == 124;  // lane 31 is the halo lane
    // u8 tensor map over 32-bit words: a strip starts at word cs * kU8Words; TMA box starts
    // must be 16-byte aligned, so with SC = 124 (93 words per strip) the box starts at the
    // word rounded down to a multiple of 4 and the row reads skip the remainder (<= 3)
    static constexpr int kU8Words = SC * 3 / 4;
    static constexpr int kU8BoxWords = 100;       // >= 3 + 96 words; 400 B (16-B multiple)
    __host__ __device__ static constexpr int u8_box_word(int cs) { return (cs * kU8Words) & ~3; }
    __host__ __device__ static constexpr int u8_skip(int cs) { return (cs * kU8Words) & 3; }
};

// HaloFn placeholder of the lane-halo layout: the core skips the lane-31 branch
struct NoHalo {
    template <class... A>
    __device__ __forceinline__ void operator()(A&...) const {}
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "HARRIS_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra HARRIS_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 4-D TMA tile load global -> shared (x = column, y = row, c = channel,
// b = image); completion is counted in bytes on `bar`.
__device__ __forceinline__ void tma_load_4d(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y,
                                            int c, int b, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(c), "r"(b), "r"(smem_u32(bar)),
        "l"(policy)
        : "memory");
}

// 3-D TMA tile load (x = inner element, y = row, z = image).
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y, int z,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- TMA stores (shared -> global, bulk-group completion) ----
// box at (x, y, z) of the output tensor map from 128-byte aligned shared memory; out-of-bounds
// parts of the box are not written (right / bottom edges need no special code)
__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* smem_src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_u32(smem_src)), "r"(x), "r"(y), "r"(z)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N bulk groups of this thread still READING their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// every bulk group of this thread complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// order this thread's generic-proxy shared-memory writes before later async-proxy reads (TMA store)
__device__ __forceinline__ void fence_proxy_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128(float* p, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__device__ __forceinline__ uint64_t l2_policy(int which) {
    uint64_t p;
    if (which == 1)
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    else if (which == 2)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// plain C++ load (ordered after mbar_wait's "memory" clobber, free to schedule
// otherwise); p must be 16-byte aligned shared memory
__device__ __forceinline__ float2 lds64(const float* p) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ float4 lds128(const float* p) {
    return *reinterpret_cast<const float4*>(p);
}

// streaming 16-byte store (output is written once, never re-read by the kernel)
// predicated form: one SETP + one predicated STG, no branch / reconvergence point
__device__ __forceinline__ void stg128_cs_if(bool pred, float* p, float a, float b, float c, float d) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n@p st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};\n}" ::"l"(p),
        "f"(a), "f"(b), "f"(c), "f"(d), "r"(int(pred))
        : "memory");
}
__device__ __forceinline__ void stg128_cs(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

// 4 floats to an 8-byte aligned address: two 8-byte streaming stores
__device__ __forceinline__ void stg64_cs(float* p, float a, float b) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void stg2x2_cs(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p + 2), "f"(c), "f"(d) : "memory");
}

// system-scope release store / acquire load (cross-GPU flags of the fused gather)
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ------------------------------------------------------------ exact arithmetic
__device__ __forceinline__ float gray_exact(float r, float g, float b) {
    float t = __fadd_rn(0.0f, __fmul_rn(kGrayR, r));
    t = __fadd_rn(t, __fmul_rn(kGrayG, g));
    return __fadd_rn(t, __fmul_rn(kGrayB, b));
}

// 9-tap accumulation from 0 in row-major order, including the zero taps
// (PAPER.md:4613-4635).  w is row-major 3x3; g0,g1,g2 are gray rows at x..x+2.
__device__ __forceinline__ float conv9_exact(const float (&w)[9], float a0, float a1, float a2, float b0,
                                             float b1, float b2, float c0, float c1, float c2) {
    float t = 0.0f;
    t = __fadd_rn(t, __fmul_rn(w[0], a0));
    t = __fadd_rn(t, __fmul_rn(w[1], a1));
    t = __fadd_rn(t, __fmul_rn(w[2], a2));
    t = __fadd_rn(t, __fmul_rn(w[3], b0));
    t = __fadd_rn(t, __fmul_rn(w[4], b1));
    t = __fadd_rn(t, __fmul_rn(w[5], b2));
    t = __fadd_rn(t, __fmul_rn(w[6], c0));
    t = __fadd_rn(t, __fmul_rn(w[7], c1));
    t = __fadd_rn(t, __fmul_rn(w[8], c2));
    return t;
}

__device__ __forceinline__ float sum9_exact(float a0, float a1, float a2, float b0, float b1, float b2,
                                            float c0, float c1, float c2) {
    float s = __fadd_rn(0.0f, a0);
    s = __fadd_rn(s, a1);
    s = __fadd_rn(s, a2);
    s = __fadd_rn(s, b0);
    s = __fadd_rn(s, b1);
    s = __fadd_rn(s, b2);
    s = __fadd_rn(s, c0);
    s = __fadd_rn(s, c1);
    s = __fadd_rn(s, c2);
    return s;
}

__device__ __forceinline__ float coarsity_exact(float sxx, float sxy, float syy, float k) {
    float det = __fsub_rn(__fmul_rn(sxx, syy), __fmul_rn(sxy, sxy));
    float tr = __fadd_rn(sxx, syy);
    return __fsub_rn(det, __fmul_rn(__fmul_rn(k, tr), tr));
}

__device__ __forceinline__ float coarsity_fast(float sxx, float sxy, float syy, float k) {
    float det = fmaf(-sxy, sxy, sxx * syy);
    float tr = sxx + syy;
    return fmaf(-k * tr, tr, det);
}

}  // namespace harris
