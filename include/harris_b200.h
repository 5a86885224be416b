/*
 * harris_b200.h — C-ABI of the fused B200 Harris corner detector.
 *
 * Drop-in for the Harris path of arXiv 2212.12035 (the Shine thesis; reference
 * at /root/reference).  The reference has no compiled Harris entry point
 * (SURVEY.md §0.1); the boundary is defined by the thesis itself:
 *
 *   - Rise type   harris : 3.(n+4).(m+4).f32 -> n.m.f32
 *     planar channel-major RGB in, valid-region output 4 smaller per dimension,
 *     no padding.
 *   - generated kernel   harris(output, n0, n1, x0, t1, t2, t3) PAPER.md:4582-4583
 *     "output parameter followed by input parameters".
 *     Fusion removes the caller-provided scratch buffers t1..t3.
 *   - host code convention  <name>_init / <name>_run / <name>_destroy over the
 *     LRA runtime; caller owns all buffers.
 *
 * Conventions
 *   - Sizes n, m are OUTPUT rows / columns; the input is (n+4) x (m+4) per channel.
 *   - All pointers passed to harris_run* are DEVICE pointers (except
 *     harris_run_host); calls are asynchronous on `cuda_stream` (a cudaStream_t,
 *     NULL = legacy default stream).  The library never allocates in harris_run*.
 *   - Return 0 on success, a negative HARRIS_ERR_* code otherwise; nothing throws
 *     across this boundary.  harris_strerror() names the code.
 *   - A ctx is immutable after harris_init except for the host-staging buffers of
 *     harris_run_host and an internally locked launch cache (tensor maps + tile plans
 *     of the last 8 call geometries, so repeated calls skip descriptor encoding and
 *     planning), so harris_run* may be called concurrently on different streams;
 *     harris_run_host must not be called concurrently on one ctx.
 *   - Element type is f32 throughout; kappa is the coarsity constant (0.04 in the
 *     thesis).
 */
#ifndef HARRIS_B200_H
#define HARRIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HARRIS_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define HARRIS_API __attribute__((visibility("default")))
#else
#define HARRIS_API
#endif

#define HARRIS_OK                       0
#define HARRIS_ERR_INVALID_ARGUMENT   (-1)  /* null pointer, bad pitch/stride, batch < 1 */
#define HARRIS_ERR_SIZE               (-2)  /* n < 1 or m < 1 (input smaller than 5x5) or too large */
#define HARRIS_ERR_ALIGNMENT          (-3)  /* explicit TMA request on unaligned data */
#define HARRIS_ERR_CUDA               (-4)  /* CUDA runtime error (see harris_last_cuda_error) */
#define HARRIS_ERR_NO_DEVICE          (-5)  /* no CUDA device / bad device ordinal */
#define HARRIS_ERR_TMA                (-6)  /* cuTensorMapEncodeTiled failed */
#define HARRIS_ERR_OUT_OF_MEMORY      (-7)
#define HARRIS_ERR_UNSUPPORTED_DEVICE (-8)  /* not an sm_100 device */

/* flags for harris_run_strided / harris_run_host */
#define HARRIS_FLAG_EXACT_ORDER   0x1u  /* SURVEY.md App. B op order, no FMA: bit-identical
                                           to oracle/harris_oracle.c oracle_harris_f32 */
#define HARRIS_FLAG_FORCE_GENERIC 0x2u  /* use the generic (non-TMA) kernel */
#define HARRIS_FLAG_FORCE_TMA     0x4u  /* fail with HARRIS_ERR_ALIGNMENT instead of falling
                                           back to the generic GPU kernel */
#define HARRIS_FLAG_PDL           0x8u  /* programmatic dependent launch: the kernel is launched
                                           while the previous kernel on the stream may still run;
                                           its prologue overlaps that kernel's tail and it waits
                                           for it (griddepcontrol.wait) before touching memory.
                                           Safe for any stream content. */
#define HARRIS_FLAG_PDL_INDEPENDENT 0x10u /* PDL without the wait before the work: the CALLER
                                           guarantees that no earlier work on the stream that may
                                           still be running writes this call's input or reads or
                                           writes its output (a stream of independent frames in
                                           distinct buffers).  Loads start at once and the kernel
                                           fills the SMs the previous one leaves; it still
                                           completes only after the previous kernel, so later
                                           stream work sees stream order. */

#define HARRIS_FLAG_BINOMIAL_WINDOW 0x20u /* Harris with the reference's binomial window
                                           weights2d = [1,2,1]^T [1,2,1] in place of the 3x3 '+'
                                           box sums ("sometimes used as part of the Harris corner
                                           detection instead of the 3x3 '+' convolution",
                                           PAPER.md:3937-3938; weights at evalref.py:114-115).
                                           Planar f32 with TMA-describable layouts runs the fused
                                           TMA kernel; every other layout / u8 the generic kernel.
                                           EXACT order: row-major sum of w*p from 0 (oracle
                                           oracle_harris_f32_window). */

/* which kernel the last harris_run* on a ctx launched */
#define HARRIS_PATH_NONE    0
#define HARRIS_PATH_TMA     1  /* K1: TMA-staged warp-strip kernel (W%4==0, aligned) */
#define HARRIS_PATH_GENERIC 2  /* K0: shared-memory tile kernel (any W, any pitch)   */
#define HARRIS_PATH_PAIR    4  /* K1p: TMA over pairs of rows, for f32 whose row pitch is 2 (mod 4)
                                      floats (e.g. 1918 or 8190 wide) with 16-byte aligned planes,
                                      and u8 whose row pitch is 8 (mod 16) bytes (e.g. 1080 wide) */
#define HARRIS_PATH_QUAD    5  /* K1q: TMA over quads of rows, for f32 with an odd row pitch and
                                      u8 whose row pitch is 4 (mod 8) bytes (e.g. 1916 wide) */
#define HARRIS_PATH_LDG     3  /* K1b / K2: the TMA kernel's engine with one bulk copy per stage
                                      row (K1b, default) or cp.async stage fills (K2), for inputs
                                      whose strides / base TMA cannot describe (f32 with W % 4 != 0
                                      or a 4-byte aligned base; u8 with 3W % 16 != 0) */

typedef struct harris_ctx harris_ctx;

/* ~ <name>_init: binds a device, caches its properties,
 * configures the kernels.  cuda_device < 0 means the current device. */
HARRIS_API int harris_init(harris_ctx** ctx, int cuda_device);

/* Options of harris_init_ex (harris_init = harris_init_ex with harris_options_default).
 * Call harris_options_default first, then set fields; struct_size guards layout growth. */
#define HARRIS_L2_EVICT_FIRST  0
#define HARRIS_L2_EVICT_NORMAL 1
#define HARRIS_L2_EVICT_LAST   2  /* default: a strip's 4-column halo sectors are re-read by its
                                     neighbouring strip (+0.6-2 % on every shape).  The input lines of
                                     a finished launch keep evict_last priority in L2 until displaced;
                                     pick EVICT_NORMAL when the caller's next kernels need the L2. */
typedef struct harris_options {
    uint32_t struct_size;  /* sizeof(harris_options) */
    int32_t l2_policy;     /* HARRIS_L2_* for the input loads of every kernel path */
    int32_t band_rows;     /* output rows per tile; 0 = the library's planner */
    int32_t pdl;           /* 1 (default): every strip-kernel launch uses programmatic dependent
                              launch with the wait (HARRIS_FLAG_PDL semantics: safe for any stream
                              content; back-to-back calls overlap launch latency); 0: plain launches */
    int32_t reserved[4];
} harris_options;

HARRIS_API void harris_options_default(harris_options* opts);
/* harris_init with options (NULL = defaults).  Developer knobs are read from the
 * environment only when HARRIS_DEV=1 (kernel configurations, tiling, L2 promotion);
 * otherwise the environment never changes the library's behaviour. */
HARRIS_API int harris_init_ex(harris_ctx** ctx, int cuda_device, const harris_options* opts);

/* ~ <name>_destroy. NULL is accepted. */
HARRIS_API void harris_destroy(harris_ctx* ctx);

/* ~ <name>_run / kernel harris(output, n0, n1, x0, ...)
 * (PAPER.md:4582-4583).  out: n x m, row pitch out_pitch >= m elements
 * (out_pitch = m+4 reproduces the thesis kernel's output layout);
 * rgb: contiguous planar 3 x (n+4) x (m+4). */
HARRIS_API int harris_run(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t n, int64_t m,
               const float* rgb, float kappa, void* cuda_stream);

/* batch contiguous images: rgb batch x 3 x (n+4) x (m+4), out batch x n x m.
 * One launch for the whole batch (image x strip grid). */
HARRIS_API int harris_run_batched(harris_ctx* ctx, float* out, int64_t n, int64_t m,
                       const float* rgb, int64_t batch, float kappa, void* cuda_stream);

/* fully strided form every other entry point reduces to.
 * input  element (b, c, y, x) at rgb[b*in_image_stride + c*in_chan_stride + y*in_pitch + x]
 * output element (b, y, x)    at out[b*out_image_stride + y*out_pitch + x]
 * A row band of a larger image is a sub-view: rgb + r0*in_pitch with the parent's
 * in_chan_stride (this is how the multi-GPU driver shards with a 4-row halo). */
HARRIS_API int harris_run_strided(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride,
                       int64_t n, int64_t m, const float* rgb, int64_t in_pitch,
                       int64_t in_chan_stride, int64_t in_image_stride, int64_t batch,
                       float kappa, uint32_t flags, void* cuda_stream);

/* A stream of independent single frames, one launch per frame, back to back (the thesis's
 * per-frame measurement, without batching them): frame k reads the
 * planar image rgbs[k] (3 x (n+4) x (m+4), row pitch in_pitch, channel stride in_chan_stride)
 * and writes outs[k] (n x m, row pitch out_pitch).  Frame 0 is launched with HARRIS_FLAG_PDL
 * (it waits for earlier stream work; HARRIS_FLAG_PDL_INDEPENDENT in flags drops that wait),
 * frames 1.. with HARRIS_FLAG_PDL_INDEPENDENT, so each frame's kernel starts on the SMs the
 * previous frame leaves.  All outs[] must be distinct and must not overlap any rgbs[]. */
HARRIS_API int harris_run_frames(harris_ctx* ctx, float* const* outs, int64_t out_pitch, int64_t n, int64_t m,
                                 const float* const* rgbs, int64_t in_pitch, int64_t in_chan_stride,
                                 int64_t frames, float kappa, uint32_t flags, void* cuda_stream);
/* the same for interleaved 8-bit RGB frames (HWC, value/255; e.g. the thesis's PNG inputs):
 * frame k at rgb8s[k] with row pitch in_pitch_bytes */
HARRIS_API int harris_run_frames_u8(harris_ctx* ctx, float* const* outs, int64_t out_pitch, int64_t n, int64_t m,
                                    const uint8_t* const* rgb8s, int64_t in_pitch_bytes, int64_t frames, float kappa,
                                    uint32_t flags, void* cuda_stream);

/* HOST buffers (pinned for full speed; pageable works).  Row bands (batch == 1) or
 * image groups are pipelined H2D -> kernel -> D2H over three streams; returns when
 * the output is in out_host.  rgb_host: batch x 3 x (n+4) x (m+4) contiguous;
 * out_host: batch x n x out_pitch. */
HARRIS_API int harris_run_host(harris_ctx* ctx, float* out_host, int64_t out_pitch, int64_t n, int64_t m,
                    const float* rgb_host, int64_t batch, float kappa, uint32_t flags);

/* Interleaved 8-bit RGB input (HWC, e.g. a decoded rgb.png):
 * byte (b, y, x, c) at rgb8[b*in_image_stride_bytes + y*in_pitch_bytes + 3*x + c],
 * value = byte / 255.0f.  The conversion is fused into the kernel's load stage
 * (3 B per input pixel from HBM instead of 12); results equal harris_run_strided on the
 * planar f32 image byte/255 (bit-for-bit with HARRIS_FLAG_EXACT_ORDER).  TMA path when
 * the base and byte strides are 16-byte aligned, generic GPU kernel otherwise. */
HARRIS_API int harris_run_u8(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride,
                             int64_t n, int64_t m, const uint8_t* rgb8, int64_t in_pitch_bytes,
                             int64_t in_image_stride_bytes, int64_t batch, float kappa, uint32_t flags,
                             void* cuda_stream);

/* host-buffer form of harris_run_u8: rgb8_host batch x (n+4) x (m+4) x 3 contiguous */
HARRIS_API int harris_run_host_u8(harris_ctx* ctx, float* out_host, int64_t out_pitch, int64_t n, int64_t m,
                                  const uint8_t* rgb8_host, int64_t batch, float kappa, uint32_t flags);

/* Separable 3x3 stencil on f32 planes (the reference's binomial
 * filter is wv = wh = {1,2,1}):
 *   out[b][y][x] = sum_j wh[j] * (sum_i wv[i] * in[b][y+i][x+j])   (vertical then horizontal)
 * in: batch x (n+2) x (m+2) at in[b*in_image_stride + y*in_pitch + x]; out: batch x n x m.
 * Same strip/TMA engine as harris_run; HARRIS_FLAG_EXACT_ORDER rounds every product
 * and sum in that order (bit-exact with the oracle). wv, wh: 3 host floats each. */
HARRIS_API int harris_stencil3x3_sep(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride,
                                     int64_t n, int64_t m, const float* in, int64_t in_pitch,
                                     int64_t in_image_stride, int64_t batch, const float* wv, const float* wh,
                                     uint32_t flags, void* cuda_stream);

/* Device synthetic-image generator used by the bench (bit-identical to
 * oracle_synth_fill): dst (p, y, x) at dst[p*dst_plane_stride + y*dst_pitch + x] =
 * value of global plane plane0+p, row row0+y of a planes x H_global x W stack.
 * dist 0: U[0,1) (24-bit), dist 1: u8/255. */
HARRIS_API int harris_synth_fill(float* dst, int64_t planes, int64_t rows, int64_t W, int64_t dst_pitch,
                      int64_t dst_plane_stride, int64_t H_global, int64_t row0, int64_t plane0,
                      uint64_t seed, int dist, void* cuda_stream);

/* Kernel-grouping design space of the thesis, for the fusion
 * ablation: each group is a separate kernel that round-trips its intermediates
 * through HBM in caller-provided scratch (the thesis's t1..t3 temporaries).
 * Groupings 1-3 without HARRIS_FLAG_EXACT_ORDER run every group as a strip-engine kernel
 * (TMA ring, register rotation, 16-byte stores) in the fused kernel's FAST arithmetic — the
 * fair fusion ablation: grouping 3 is bit-identical to the fused FAST output, groupings 1-2
 * round the products they materialise (within tolerance); needs W % 4 == 0 and 16-byte
 * aligned buffers.  With HARRIS_FLAG_EXACT_ORDER (or other layouts) the groups are simple
 * one-thread-per-pixel kernels in the Appendix-B order (bit-identical to the oracle).
 * Grouping 4 is harris_run_strided (flags honoured).  Contiguous single image. */
#define HARRIS_GROUPING_UNFUSED    1  /* [Sx],[Sy],[x],[+],[coarsity]  5 kernels */
#define HARRIS_GROUPING_SOBEL_PROD 2  /* [Sx,Sy,x],[+,coarsity]        2 kernels */
#define HARRIS_GROUPING_SOBEL      3  /* [Sx,Sy],[x,+,coarsity]        2 kernels */
#define HARRIS_GROUPING_FUSED      4  /* [Sx,Sy,x,+,coarsity]          1 kernel  */

HARRIS_API int64_t harris_grouping_scratch_bytes(int grouping, int64_t n, int64_t m);
HARRIS_API int harris_grouping_launches(int grouping);
HARRIS_API int harris_run_grouping(harris_ctx* ctx, int grouping, float* out, int64_t n, int64_t m,
                                   const float* rgb, void* scratch, int64_t scratch_bytes, float kappa,
                                   uint32_t flags, void* cuda_stream);

/* ---- fused gather over peer memory ("results gathered over NVLink only
 * for the final output").  The root exports its result buffer and a flag array
 * (one uint32 slot per rank); every rank maps both (CUDA IPC; NVLink 5 / NVSwitch P2P on
 * a multi-GPU node) and calls harris_run_notify with `out` pointing at its rows / images
 * inside the root's buffer: the fused kernel's output stores travel over the link as
 * each row is produced, and its last CTA releases `epoch` into the rank's flag slot.
 * The root enqueues harris_peer_wait on its stream; work queued after it sees the whole
 * result.  No host barrier and no collective call in the data path. */
typedef struct harris_peer_handle {
    unsigned char ipc[64];  /* cudaIpcMemHandle_t of the allocation holding the pointer */
    int64_t offset;         /* byte offset of the exported pointer inside the allocation */
    int64_t bytes;          /* bytes from the exported pointer to the end of the allocation */
    int32_t device;         /* exporting device ordinal */
    int32_t reserved;
} harris_peer_handle;

/* export a device pointer (any address inside a cudaMalloc allocation) for other processes */
HARRIS_API int harris_peer_export(const void* dev_ptr, harris_peer_handle* out);
/* map an exported pointer on `cuda_device` (another process; peer access enabled lazily).
 * *ptr = the exported address in this process; *mapping is what harris_peer_close takes. */
HARRIS_API int harris_peer_open(int cuda_device, const harris_peer_handle* h, void** mapping, void** ptr);
HARRIS_API int harris_peer_close(int cuda_device, void* mapping);

/* harris_run_strided + completion notification: after every CTA's output stores are
 * performed at system scope, the kernel's last CTA stores `epoch` to *notify_flag with
 * release semantics (system scope).  notify_flag may be a peer mapping.  Calls with a
 * notify flag must not run concurrently on one ctx (they share its CTA counter). */
HARRIS_API int harris_run_notify(harris_ctx* ctx, float* out, int64_t out_pitch, int64_t out_image_stride,
                                 int64_t n, int64_t m, const float* rgb, int64_t in_pitch,
                                 int64_t in_chan_stride, int64_t in_image_stride, int64_t batch, float kappa,
                                 uint32_t flags, uint32_t* notify_flag, uint32_t epoch, void* cuda_stream);
/* store `epoch` to *flag (release, system scope) once earlier work on the stream is done
 * (for a rank that owns no rows) */
HARRIS_API int harris_peer_signal(uint32_t* flag, uint32_t epoch, void* cuda_stream);
/* stream-ordered wait until every flags[i] >= epoch (modular); gives up after timeout_ns
 * (<= 0: never) and then ORs 1 into *status (device memory, may be NULL) */
HARRIS_API int harris_peer_wait(const uint32_t* flags, int32_t count, uint32_t epoch, uint32_t* status,
                                int64_t timeout_ns, void* cuda_stream);

/* Launch geometry the TMA kernel would use (for tests / bench reporting). */
typedef struct harris_plan_info {
    int32_t path;           /* HARRIS_PATH_* that harris_run_strided would take */
    int32_t warps_per_cta;
    int32_t stages;
    int32_t rows_per_stage;
    int64_t band_rows;      /* output rows per tile */
    int64_t bands;          /* tiles per image column */
    int64_t col_segments;   /* warp strips per image row (strip_cols columns each) */
    int64_t tiles;          /* batch * bands * col_segments */
    int64_t grid_ctas;
    int64_t smem_bytes;     /* dynamic shared memory per CTA */
    int32_t groups;         /* 128-column strips per tile (2: packed FP32x2 dual-strip core) */
    int32_t tma_config;     /* kernel configuration index (HARRIS_TMA_CONFIG) */
    int32_t strip_cols;     /* output columns per strip (128, or 124 with the lane-halo layout) */
    int32_t reserved;
} harris_plan_info;

HARRIS_API int harris_plan(harris_ctx* ctx, int64_t n, int64_t m, int64_t batch, const float* rgb,
                int64_t in_pitch, int64_t in_chan_stride, int64_t in_image_stride,
                const float* out, int64_t out_pitch, int64_t out_image_stride,
                uint32_t flags, harris_plan_info* info);

HARRIS_API int harris_last_path(const harris_ctx* ctx);
HARRIS_API int harris_device(const harris_ctx* ctx);
HARRIS_API int harris_num_sms(const harris_ctx* ctx);
HARRIS_API const char* harris_strerror(int code);
HARRIS_API const char* harris_last_cuda_error(const harris_ctx* ctx);
HARRIS_API int harris_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HARRIS_B200_H */
