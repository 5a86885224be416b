// harris_groupings.cu — the thesis's kernel-grouping design space on B200
// (Table "Four different kernel
// groupings"):
//
//   1  [Sx], [Sy], [x], [+], [coarsity]      5 kernels, intermediates in HBM
//   2  [Sx, Sy, x], [+, coarsity]            2 kernels
//   3  [Sx, Sy], [x, +, coarsity]            2 kernels
//   4  [Sx, Sy, x, +, coarsity]              1 kernel  (= harris_run, the TMA kernel)
//
// Grayscale is recomputed inside every Sobel group, as in the thesis (gray is a
// pointwise producer fused into its consumers).  Each group reads its inputs
// from and writes its outputs to HBM through caller-provided scratch (the
// thesis's t1..t3 temporaries), so the groupings quantify
// what operator fusion saves in HBM bytes on this machine.  Every stage uses the
// Appendix-B op order (harris_common.cuh), so every grouping is bit-identical to
// the C oracle — the ablation changes traffic, never results.
//
// These kernels are deliberately simple (one thread per pixel, coalesced rows,
// stencil neighbours through L1): they are the unfused baseline, not the product.
#include <cuda_runtime.h>

#include <cstdint>

#include "harris_common.cuh"
#include "harris_internal.h"

namespace harris {

namespace {

constexpr int kBX = 128, kBY = 2;

__constant__ float cWX[9] = {-kSobA, 0.f, kSobA, -kSobB, 0.f, kSobB, -kSobA, 0.f, kSobA};
__constant__ float cWY[9] = {-kSobA, -kSobB, -kSobA, 0.f, 0.f, 0.f, kSobA, kSobB, kSobA};

struct Planes {
    int64_t H, W;  // input
};

__device__ __forceinline__ float gray_at(const float* __restrict__ rgb, int64_t HW, int64_t W, int64_t y,
                                         int64_t x) {
    const float* p = rgb + y * W + x;
    return gray_exact(__ldg(p), __ldg(p + HW), __ldg(p + 2 * HW));
}

// Sobel group: gray recomputed for the 3x3 window; writes Ix and/or Iy and/or products.
template <bool WX, bool WY, bool PROD>
__global__ void __launch_bounds__(kBX* kBY) k_sobel(const float* __restrict__ rgb, int64_t H, int64_t W,
                                                     float* __restrict__ ix_out, float* __restrict__ iy_out,
                                                     float* __restrict__ pxx, float* __restrict__ pxy,
                                                     float* __restrict__ pyy) {
    const int64_t Hs = H - 2, Ws = W - 2;
    const int64_t x = int64_t(blockIdx.x) * kBX + threadIdx.x;
    const int64_t y = int64_t(blockIdx.y) * kBY + threadIdx.y;
    if (x >= Ws || y >= Hs) return;
    const int64_t HW = H * W;
    float g[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) g[3 * i + j] = gray_at(rgb, HW, W, y + i, x + j);
    float ix = 0.f, iy = 0.f;
    if (WX || PROD) ix = conv9_exact(cWX, g[0], g[1], g[2], g[3], g[4], g[5], g[6], g[7], g[8]);
    if (WY || PROD) iy = conv9_exact(cWY, g[0], g[1], g[2], g[3], g[4], g[5], g[6], g[7], g[8]);
    const int64_t o = y * Ws + x;
    if (PROD) {
        pxx[o] = __fmul_rn(ix, ix);
        pxy[o] = __fmul_rn(ix, iy);
        pyy[o] = __fmul_rn(iy, iy);
    } else {
        if (WX) ix_out[o] = ix;
        if (WY) iy_out[o] = iy;
    }
}

__global__ void __launch_bounds__(kBX* kBY) k_products(const float* __restrict__ ix, const float* __restrict__ iy,
                                                        int64_t count, float* __restrict__ pxx,
                                                        float* __restrict__ pxy, float* __restrict__ pyy) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x * blockDim.y + threadIdx.y * blockDim.x + threadIdx.x;
         i < count; i += int64_t(gridDim.x) * blockDim.x * blockDim.y) {
        const float a = ix[i], b = iy[i];
        pxx[i] = __fmul_rn(a, a);
        pxy[i] = __fmul_rn(a, b);
        pyy[i] = __fmul_rn(b, b);
    }
}

__device__ __forceinline__ float box9(const float* __restrict__ p, int64_t Ws, int64_t y, int64_t x) {
    const float* r0 = p + y * Ws + x;
    const float* r1 = r0 + Ws;
    const float* r2 = r1 + Ws;
    return sum9_exact(__ldg(r0), __ldg(r0 + 1), __ldg(r0 + 2), __ldg(r1), __ldg(r1 + 1), __ldg(r1 + 2), __ldg(r2),
                      __ldg(r2 + 1), __ldg(r2 + 2));
}

// [+] alone (COARS=false: writes S**) or [+, coarsity] (COARS=true: writes out)
template <bool COARS>
__global__ void __launch_bounds__(kBX* kBY) k_box(const float* __restrict__ pxx, const float* __restrict__ pxy,
                                                   const float* __restrict__ pyy, int64_t n, int64_t m,
                                                   float* __restrict__ sxx, float* __restrict__ sxy,
                                                   float* __restrict__ syy, float* __restrict__ out, float kappa) {
    const int64_t x = int64_t(blockIdx.x) * kBX + threadIdx.x;
    const int64_t y = int64_t(blockIdx.y) * kBY + threadIdx.y;
    if (x >= m || y >= n) return;
    const int64_t Ws = m + 2;
    const float a = box9(pxx, Ws, y, x), b = box9(pxy, Ws, y, x), c = box9(pyy, Ws, y, x);
    const int64_t o = y * m + x;
    if (COARS) {
        out[o] = coarsity_exact(a, b, c, kappa);
    } else {
        sxx[o] = a;
        sxy[o] = b;
        syy[o] = c;
    }
}

__global__ void __launch_bounds__(kBX* kBY) k_coarsity(const float* __restrict__ sxx, const float* __restrict__ sxy,
                                                        const float* __restrict__ syy, int64_t count,
                                                        float* __restrict__ out, float kappa) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x * blockDim.y + threadIdx.y * blockDim.x + threadIdx.x;
         i < count; i += int64_t(gridDim.x) * blockDim.x * blockDim.y)
        out[i] = coarsity_exact(sxx[i], sxy[i], syy[i], kappa);
}

// [x, +, coarsity]: products recomputed per box tap (exactly representable: the
// product of two f32 is rounded identically wherever it is computed)
__global__ void __launch_bounds__(kBX* kBY) k_prod_box_coarsity(const float* __restrict__ ix,
                                                                 const float* __restrict__ iy, int64_t n,
                                                                 int64_t m, float* __restrict__ out, float kappa) {
    const int64_t x = int64_t(blockIdx.x) * kBX + threadIdx.x;
    const int64_t y = int64_t(blockIdx.y) * kBY + threadIdx.y;
    if (x >= m || y >= n) return;
    const int64_t Ws = m + 2;
    float a[9], b[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            a[3 * i + j] = __ldg(ix + (y + i) * Ws + x + j);
            b[3 * i + j] = __ldg(iy + (y + i) * Ws + x + j);
        }
    float pxx[9], pxy[9], pyy[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        pxx[k] = __fmul_rn(a[k], a[k]);
        pxy[k] = __fmul_rn(a[k], b[k]);
        pyy[k] = __fmul_rn(b[k], b[k]);
    }
    const float sxx = sum9_exact(pxx[0], pxx[1], pxx[2], pxx[3], pxx[4], pxx[5], pxx[6], pxx[7], pxx[8]);
    const float sxy = sum9_exact(pxy[0], pxy[1], pxy[2], pxy[3], pxy[4], pxy[5], pxy[6], pxy[7], pxy[8]);
    const float syy = sum9_exact(pyy[0], pyy[1], pyy[2], pyy[3], pyy[4], pyy[5], pyy[6], pyy[7], pyy[8]);
    out[y * m + x] = coarsity_exact(sxx, sxy, syy, kappa);
}

inline dim3 grid2d(int64_t cols, int64_t rows) {
    return dim3(unsigned((cols + kBX - 1) / kBX), unsigned((rows + kBY - 1) / kBY));
}

inline unsigned grid1d(int64_t count, int num_sms) {
    const int64_t want = (count + kBX * kBY - 1) / (kBX * kBY);
    const int64_t cap = int64_t(num_sms) * 8;
    return unsigned(want < cap ? want : cap);
}

}  // namespace

int64_t grouping_scratch_floats(int grouping, int64_t n, int64_t m) {
    const int64_t s = (n + 2) * (m + 2), o = n * m;
    switch (grouping) {
        case 1: return 2 * s + 3 * s + 3 * o;  // Ix, Iy, products, sums
        case 2: return 3 * s;                  // products
        case 3: return 2 * s;                  // Ix, Iy
        case 4: return 0;
        default: return -1;
    }
}

int grouping_launches(int grouping) {
    switch (grouping) {
        case 1: return 5;
        case 2: case 3: return 2;
        case 4: return 1;
        default: return 0;
    }
}

cudaError_t launch_grouping(int grouping, float* out, int64_t n, int64_t m, const float* rgb, float* scratch,
                            float kappa, int num_sms, cudaStream_t st) {
    const int64_t H = n + 4, W = m + 4, Hs = n + 2, Ws = m + 2;
    const int64_t s = Hs * Ws, o = n * m;
    const dim3 blk(kBX, kBY);
    switch (grouping) {
        case 1: {
            float *ix = scratch, *iy = ix + s, *pxx = iy + s, *pxy = pxx + s, *pyy = pxy + s;
            float *sxx = pyy + s, *sxy = sxx + o, *syy = sxy + o;
            k_sobel<true, false, false><<<grid2d(Ws, Hs), blk, 0, st>>>(rgb, H, W, ix, nullptr, nullptr, nullptr,
                                                                        nullptr);
            k_sobel<false, true, false><<<grid2d(Ws, Hs), blk, 0, st>>>(rgb, H, W, nullptr, iy, nullptr, nullptr,
                                                                        nullptr);
            k_products<<<grid1d(s, num_sms), blk, 0, st>>>(ix, iy, s, pxx, pxy, pyy);
            k_box<false><<<grid2d(m, n), blk, 0, st>>>(pxx, pxy, pyy, n, m, sxx, sxy, syy, nullptr, kappa);
            k_coarsity<<<grid1d(o, num_sms), blk, 0, st>>>(sxx, sxy, syy, o, out, kappa);
            break;
        }
        case 2: {
            float *pxx = scratch, *pxy = pxx + s, *pyy = pxy + s;
            k_sobel<false, false, true><<<grid2d(Ws, Hs), blk, 0, st>>>(rgb, H, W, nullptr, nullptr, pxx, pxy, pyy);
            k_box<true><<<grid2d(m, n), blk, 0, st>>>(pxx, pxy, pyy, n, m, nullptr, nullptr, nullptr, out, kappa);
            break;
        }
        case 3: {
            float *ix = scratch, *iy = ix + s;
            k_sobel<true, true, false><<<grid2d(Ws, Hs), blk, 0, st>>>(rgb, H, W, ix, iy, nullptr, nullptr, nullptr);
            k_prod_box_coarsity<<<grid2d(m, n), blk, 0, st>>>(ix, iy, n, m, out, kappa);
            break;
        }
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace harris
