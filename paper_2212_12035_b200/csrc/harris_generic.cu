// harris_generic.cu — K0: generic fused Harris kernel (any width, any pitch,
// any alignment).  Used when the TMA kernel's constraints (16-byte aligned rows
// and strides) do not hold; it is still the fused GPU path, never a CPU one.
//
// Classic staged shared-memory stencil: a CTA owns a 32x32 output tile; it
// builds the 36x36 gray tile from coalesced scalar loads, then the 34x34 Ix/Iy
// tiles and their products, then the 3x3 box sums and coarsity, all in shared
// memory (nothing intermediate reaches HBM).  Same EXACT/FAST arithmetic
// contract as harris_tma.cu (see harris_common.cuh).
#include <cuda_runtime.h>

#include <cstdint>

#include "harris_common.cuh"
#include "harris_internal.h"

namespace harris {

constexpr int kGT = 32;          // output tile edge
constexpr int kGG = kGT + 4;     // gray tile edge
constexpr int kGS = kGT + 2;     // Sobel / product tile edge
constexpr int kGThreadsX = 32, kGThreadsY = 8;

// U8: interleaved RGB bytes (HWC), value/255; Geom.rgb is the byte base pointer and
// in_pitch / in_image_stride are byte strides.
template <bool EXACT, bool U8>
__global__ void __launch_bounds__(kGThreadsX* kGThreadsY)
    harris_generic_kernel(const Geom g, int tiles_x, int tiles_y) {
    __shared__ float gs[kGG][kGG + 1];
    __shared__ float pxx[kGS][kGS + 1], pxy[kGS][kGS + 1], pyy[kGS][kGS + 1];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * kGThreadsX + tx;
    const int nthreads = kGThreadsX * kGThreadsY;
    const int64_t H = g.n + 4, W = g.m + 4;
    const int64_t tiles = int64_t(tiles_x) * tiles_y;
    const float WX[9] = {-kSobA, 0.f, kSobA, -kSobB, 0.f, kSobB, -kSobA, 0.f, kSobA};
    const float WY[9] = {-kSobA, -kSobB, -kSobA, 0.f, 0.f, 0.f, kSobA, kSobB, kSobA};
    const float W2D[9] = {1.f, 2.f, 1.f, 2.f, 4.f, 2.f, 1.f, 2.f, 1.f};

    for (int64_t b = blockIdx.z; b < g.batch; b += gridDim.z) {
        const float* img = U8 ? g.rgb : g.rgb + b * g.in_image_stride;
        const uint8_t* img8 = reinterpret_cast<const uint8_t*>(g.rgb) + (U8 ? b * g.in_image_stride : 0);
        float* out = g.out + b * g.out_image_stride;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int64_t y0 = (t / tiles_x) * kGT, x0 = (t % tiles_x) * kGT;
            __syncthreads();  // previous tile's readers are done
            for (int e = tid; e < kGG * kGG; e += nthreads) {
                const int yy = e / kGG, xx = e % kGG;
                const int64_t y = y0 + yy, x = x0 + xx;
                float v = 0.f;
                if (y < H && x < W) {
                    float r, gr, bl;
                    if (U8) {
                        const uint8_t* p = img8 + y * g.in_pitch + 3 * x;
                        r = __fdiv_rn(float(__ldg(p)), 255.0f);
                        gr = __fdiv_rn(float(__ldg(p + 1)), 255.0f);
                        bl = __fdiv_rn(float(__ldg(p + 2)), 255.0f);
                    } else {
                        const float* p = img + y * g.in_pitch + x;
                        r = __ldg(p);
                        gr = __ldg(p + g.in_chan_stride);
                        bl = __ldg(p + 2 * g.in_chan_stride);
                    }
                    v = EXACT ? gray_exact(r, gr, bl) : fmaf(kGrayB, bl, fmaf(kGrayG, gr, kGrayR * r));
                }
                gs[yy][xx] = v;
            }
            __syncthreads();
            for (int e = tid; e < kGS * kGS; e += nthreads) {
                const int yy = e / kGS, xx = e % kGS;
                float ix, iy;
                if (EXACT) {
                    ix = conv9_exact(WX, gs[yy][xx], gs[yy][xx + 1], gs[yy][xx + 2], gs[yy + 1][xx],
                                     gs[yy + 1][xx + 1], gs[yy + 1][xx + 2], gs[yy + 2][xx], gs[yy + 2][xx + 1],
                                     gs[yy + 2][xx + 2]);
                    iy = conv9_exact(WY, gs[yy][xx], gs[yy][xx + 1], gs[yy][xx + 2], gs[yy + 1][xx],
                                     gs[yy + 1][xx + 1], gs[yy + 1][xx + 2], gs[yy + 2][xx], gs[yy + 2][xx + 1],
                                     gs[yy + 2][xx + 2]);
                    pxx[yy][xx] = __fmul_rn(ix, ix);
                    pxy[yy][xx] = __fmul_rn(ix, iy);
                    pyy[yy][xx] = __fmul_rn(iy, iy);
                } else {
                    const float d0 = gs[yy][xx + 2] - gs[yy][xx];
                    const float d1 = gs[yy + 1][xx + 2] - gs[yy + 1][xx];
                    const float d2 = gs[yy + 2][xx + 2] - gs[yy + 2][xx];
                    const float h0 = fmaf(2.f, gs[yy][xx + 1], gs[yy][xx]) + gs[yy][xx + 2];
                    const float h2 = fmaf(2.f, gs[yy + 2][xx + 1], gs[yy + 2][xx]) + gs[yy + 2][xx + 2];
                    ix = kSobA * fmaf(2.f, d1, d0 + d2);
                    iy = kSobA * (h2 - h0);
                    pxx[yy][xx] = ix * ix;
                    pxy[yy][xx] = ix * iy;
                    pyy[yy][xx] = iy * iy;
                }
            }
            __syncthreads();
            for (int e = tid; e < kGT * kGT; e += nthreads) {
                const int yy = e / kGT, xx = e % kGT;
                const int64_t y = y0 + yy, x = x0 + xx;
                if (y >= g.n || x >= g.m) continue;
                float s[3];
                float(*pp[3])[kGS + 1] = {pxx, pxy, pyy};
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    float(*p)[kGS + 1] = pp[q];
                    if (g.window) {  // binomial window (HARRIS_FLAG_BINOMIAL_WINDOW)
                        if (EXACT) {
                            s[q] = conv9_exact(W2D, p[yy][xx], p[yy][xx + 1], p[yy][xx + 2], p[yy + 1][xx],
                                               p[yy + 1][xx + 1], p[yy + 1][xx + 2], p[yy + 2][xx], p[yy + 2][xx + 1],
                                               p[yy + 2][xx + 2]);
                        } else {
                            float c[3];
#pragma unroll
                            for (int j = 0; j < 3; ++j)
                                c[j] = fmaf(2.f, p[yy + 1][xx + j], p[yy][xx + j] + p[yy + 2][xx + j]);
                            s[q] = fmaf(2.f, c[1], c[0] + c[2]);
                        }
                    } else if (EXACT) {
                        s[q] = sum9_exact(p[yy][xx], p[yy][xx + 1], p[yy][xx + 2], p[yy + 1][xx], p[yy + 1][xx + 1],
                                          p[yy + 1][xx + 2], p[yy + 2][xx], p[yy + 2][xx + 1], p[yy + 2][xx + 2]);
                    } else {
                        s[q] = (p[yy][xx] + p[yy + 1][xx] + p[yy + 2][xx]) +
                               (p[yy][xx + 1] + p[yy + 1][xx + 1] + p[yy + 2][xx + 1]) +
                               (p[yy][xx + 2] + p[yy + 1][xx + 2] + p[yy + 2][xx + 2]);
                    }
                }
                out[y * g.out_pitch + x] =
                    EXACT ? coarsity_exact(s[0], s[1], s[2], g.kappa) : coarsity_fast(s[0], s[1], s[2], g.kappa);
            }
        }
    }
}

template <bool U8>
static cudaError_t launch_generic_t(bool exact, const Geom& g, cudaStream_t stream) {
    const int tiles_x = int((g.m + kGT - 1) / kGT), tiles_y = int((g.n + kGT - 1) / kGT);
    const int64_t tiles = int64_t(tiles_x) * tiles_y;
    const dim3 block{kGThreadsX, kGThreadsY, 1};
    const unsigned gx = unsigned(tiles < 65535 * 8 ? tiles : 65535 * 8);
    const unsigned gz = unsigned(g.batch < 65535 ? g.batch : 65535);
    const dim3 grid{gx, 1, gz};
    if (exact)
        harris_generic_kernel<true, U8><<<grid, block, 0, stream>>>(g, tiles_x, tiles_y);
    else
        harris_generic_kernel<false, U8><<<grid, block, 0, stream>>>(g, tiles_x, tiles_y);
    return cudaGetLastError();
}

cudaError_t launch_generic(bool exact, const Geom& g, cudaStream_t stream) {
    return launch_generic_t<false>(exact, g, stream);
}

cudaError_t launch_generic_u8(bool exact, const Geom& g, cudaStream_t stream) {
    return launch_generic_t<true>(exact, g, stream);
}

}  // namespace harris
