// harris_synth.cu — device synthetic planar-RGB generator for the bench and the
// multi-GPU driver.  Every element is mix64(global linear index + seed*K)
// (splitmix64 finaliser), so any row band of any plane regenerates identically
// on any device and on the host (oracle_synth_fill / oracle.synth.synth_numpy
// are bit-exact mirrors used by the tests).  HBM-write-bound: one float4 store
// per thread iteration, grid-stride over a multiple of the SM count.
#include <cuda_runtime.h>

#include <cstdint>

#include "harris_internal.h"

namespace harris {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float synth_value(uint64_t idx, uint64_t key, int dist) {
    const uint64_t z = mix64(idx + key);
    return dist == 1 ? __fdiv_rn(float(z >> 56), 255.0f) : float(z >> 40) * 0x1p-24f;
}

__global__ void synth_kernel(float* __restrict__ dst, int64_t planes, int64_t rows, int64_t W, int64_t dst_pitch,
                             int64_t dst_plane_stride, int64_t H_global, int64_t row0, int64_t plane0,
                             uint64_t key, int dist) {
    const int64_t qpr = (W + 3) / 4;  // float4 quads per row
    const int64_t total = planes * rows * qpr;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = e % qpr;
        const int64_t pr = e / qpr;
        const int64_t y = pr % rows, p = pr / rows;
        const int64_t x = q * 4;
        const uint64_t base = (uint64_t(plane0 + p) * uint64_t(H_global) + uint64_t(row0 + y)) * uint64_t(W);
        float* row = dst + p * dst_plane_stride + y * dst_pitch;
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = synth_value(base + uint64_t(x + k), key, dist);
        const bool vec = (x + 4 <= W) && ((reinterpret_cast<uintptr_t>(row + x) & 15) == 0);
        if (vec) {
            *reinterpret_cast<float4*>(row + x) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
            for (int k = 0; k < 4 && x + k < W; ++k) row[x + k] = v[k];
        }
    }
}

cudaError_t launch_synth(float* dst, int64_t planes, int64_t rows, int64_t W, int64_t dst_pitch,
                         int64_t dst_plane_stride, int64_t H_global, int64_t row0, int64_t plane0, uint64_t seed,
                         int dist, int num_sms, cudaStream_t stream) {
    const int64_t total = planes * rows * ((W + 3) / 4);
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = int64_t(num_sms > 0 ? num_sms : 148) * 16;
    if (blocks > cap) blocks = cap;
    const uint64_t key = seed * 0xD1B54A32D192ED03ull;
    synth_kernel<<<unsigned(blocks), 256, 0, stream>>>(dst, planes, rows, W, dst_pitch, dst_plane_stride, H_global,
                                                      row0, plane0, key, dist);
    return cudaGetLastError();
}

}  // namespace harris
