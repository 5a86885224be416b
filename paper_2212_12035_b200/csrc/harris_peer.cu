// harris_peer.cu — peer-memory plumbing of the fused gather (
// BASELINE.json north_star: "results are gathered over NVLink only for the final
// output").
//
// The gather is not a separate collective: every rank runs the fused Harris kernel
// with its output pointer aimed straight into the root's result buffer (a CUDA IPC
// mapping of the root's allocation — NVLink 5 / NVSwitch P2P stores on a multi-GPU
// node), so each output row crosses the link as soon as it is computed and the
// transfer overlaps the rest of the stencil.  The kernel's last CTA then releases an
// epoch into the rank's slot of a flag array in the root's memory
// (strip_pipeline.cuh notify_epilogue); the root's stream acquires every slot with a
// one-warp spin kernel (peer_wait_kernel) before anything downstream reads the result.
// No host barrier and no NCCL call sits in the data path.
//
// This file: the IPC export/open/close entry points and the standalone
// signal / wait kernels (the signal kernel serves ranks whose launch went through the
// generic kernel or that own no rows).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstring>

#include "../../include/harris_b200.h"
#include "harris_common.cuh"
#include "harris_internal.h"

namespace harris {

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void peer_signal_kernel(uint32_t* flag, uint32_t epoch) {
    // everything earlier on this stream (the producer kernel's peer stores) has completed;
    // the system-scope fence + release store publish it to the consumer GPU
    __threadfence_system();
    st_release_sys(flag, epoch);
}

// One thread per flag slot: spin (acquire, system scope) until slot >= epoch (modular
// comparison, epochs wrap), or give up after timeout_ns and raise bit 0 of *status so a
// dead peer can never hang the consumer GPU.
__global__ void peer_wait_kernel(const uint32_t* flags, int32_t count, uint32_t epoch, uint32_t* status,
                                 int64_t timeout_ns) {
    const uint64_t t0 = globaltimer_ns();
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        uint32_t sleep_ns = 32;
        while (int32_t(ld_acquire_sys(flags + i) - epoch) < 0) {
            if (timeout_ns > 0 && int64_t(globaltimer_ns() - t0) > timeout_ns) {
                if (status) atomicOr(status, 1u);
                break;
            }
            __nanosleep(sleep_ns);
            if (sleep_ns < 1024) sleep_ns <<= 1;
        }
    }
    __syncthreads();
    __threadfence_system();  // order the acquires before anything later on this stream
}

cudaError_t launch_peer_signal(uint32_t* flag, uint32_t epoch, cudaStream_t stream) {
    peer_signal_kernel<<<1, 1, 0, stream>>>(flag, epoch);
    return cudaGetLastError();
}

cudaError_t launch_peer_wait(const uint32_t* flags, int32_t count, uint32_t epoch, uint32_t* status,
                             int64_t timeout_ns, cudaStream_t stream) {
    const int threads = count <= 32 ? 32 : (count <= 1024 ? ((count + 31) / 32) * 32 : 1024);
    peer_wait_kernel<<<1, threads, 0, stream>>>(flags, count, epoch, status, timeout_ns);
    return cudaGetLastError();
}

}  // namespace harris

namespace {

struct PeerDeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit PeerDeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (dev >= 0 && prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~PeerDeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int peer_cuda_fail(cudaError_t e) {
    cudaGetLastError();  // clear the sticky-free error state of the runtime
    return e == cudaErrorMemoryAllocation ? HARRIS_ERR_OUT_OF_MEMORY : HARRIS_ERR_CUDA;
}

PFN_cuMemGetAddressRange_v3020 address_range_fn() {
    static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
    }
    return fn;
}

}  // namespace

extern "C" {

int harris_peer_export(const void* dev_ptr, harris_peer_handle* out) {
    if (!dev_ptr || !out) return HARRIS_ERR_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof(*out));
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, dev_ptr);
    if (e != cudaSuccess) return peer_cuda_fail(e);
    if (attr.type != cudaMemoryTypeDevice) return HARRIS_ERR_INVALID_ARGUMENT;
    PeerDeviceGuard guard(attr.device);
    if (!guard.ok) return peer_cuda_fail(cudaGetLastError());
    // the IPC handle names the whole allocation; record where dev_ptr sits inside it
    auto range = address_range_fn();
    if (!range) return HARRIS_ERR_CUDA;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return HARRIS_ERR_CUDA;
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return peer_cuda_fail(e);
    static_assert(sizeof(h) <= sizeof(out->ipc), "cudaIpcMemHandle_t size");
    std::memcpy(out->ipc, &h, sizeof(h));
    out->offset = int64_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    out->bytes = int64_t(size) - out->offset;
    out->device = attr.device;
    return HARRIS_OK;
}

int harris_peer_open(int cuda_device, const harris_peer_handle* h, void** mapping, void** ptr) {
    if (!h || !mapping || !ptr || h->offset < 0 || h->bytes < 0) return HARRIS_ERR_INVALID_ARGUMENT;
    *mapping = nullptr;
    *ptr = nullptr;
    PeerDeviceGuard guard(cuda_device);
    if (!guard.ok) return HARRIS_ERR_NO_DEVICE;
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, h->ipc, sizeof(ih));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return peer_cuda_fail(e);
    *mapping = base;
    *ptr = static_cast<unsigned char*>(base) + h->offset;
    return HARRIS_OK;
}

int harris_peer_close(int cuda_device, void* mapping) {
    if (!mapping) return HARRIS_OK;
    PeerDeviceGuard guard(cuda_device);
    if (!guard.ok) return HARRIS_ERR_NO_DEVICE;
    cudaError_t e = cudaIpcCloseMemHandle(mapping);
    return e == cudaSuccess ? HARRIS_OK : peer_cuda_fail(e);
}

int harris_peer_signal(uint32_t* flag, uint32_t epoch, void* cuda_stream) {
    if (!flag) return HARRIS_ERR_INVALID_ARGUMENT;
    cudaError_t e = harris::launch_peer_signal(flag, epoch, static_cast<cudaStream_t>(cuda_stream));
    return e == cudaSuccess ? HARRIS_OK : peer_cuda_fail(e);
}

int harris_peer_wait(const uint32_t* flags, int32_t count, uint32_t epoch, uint32_t* status, int64_t timeout_ns,
                     void* cuda_stream) {
    if (count < 0 || (count > 0 && !flags)) return HARRIS_ERR_INVALID_ARGUMENT;
    if (count == 0) return HARRIS_OK;
    cudaError_t e =
        harris::launch_peer_wait(flags, count, epoch, status, timeout_ns, static_cast<cudaStream_t>(cuda_stream));
    return e == cudaSuccess ? HARRIS_OK : peer_cuda_fail(e);
}

}  // extern "C"
