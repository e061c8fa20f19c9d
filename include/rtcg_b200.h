/*
 * rtcg_b200.h -- C ABI of the B200 run-time code generation runtime
 * (librtcg_b200.so, built from paper_0911_3456_b200/csrc/rtcg_runtime.cpp).
 *
 * The reference toolkit (rtcg-kit, /root/reference/pkg/src/rtcg) compiles
 * generated C with the host `cc` and calls it through ctypes with the fixed
 * ABI `void name(void **args, long start, long end)`.  This library is the
 * drop-in replacement for the three native seams of that path:
 *
 *   compile backend   jit._run_compiler            src/jit.py:446-474
 *   module loading    jit._load_library             src/jit.py:439-443
 *   symbol lookup     jit.get_kernel                src/jit.py:557-564
 *   kernel call       jit.KernelHandle.__call__     src/jit.py:553-554
 *   storage           ndarray._system_alloc         src/ndarray.py:158-160
 *   zero on reuse     ctypes.memset in MemoryPool   src/ndarray.py:216
 *   host transfers    NdArray.to_host/copy_from_host src/ndarray.py:316-336
 *
 * Every entry point returns an int status (RTCG_OK == 0) and, on failure,
 * leaves a message retrievable with rtcg_last_error() on the calling thread.
 * No CUDA or torch types appear in the signatures: device pointers are
 * uint64_t, modules / functions / streams / events are opaque handles.
 *
 * libcuda.so.1 and libnvrtc.so.12 are loaded lazily with dlopen, so the
 * library loads (and NVRTC compiles) on hosts without a GPU; driver calls then
 * fail with RTCG_ERR_NO_DEVICE.
 */
#ifndef RTCG_B200_H
#define RTCG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTCG_ABI_VERSION 1

enum rtcg_status {
    RTCG_OK = 0,
    RTCG_ERR_CUDA = 1,          /* any other driver error                     */
    RTCG_ERR_OUT_OF_MEMORY = 2, /* CUDA_ERROR_OUT_OF_MEMORY (pool retries)     */
    RTCG_ERR_NOT_FOUND = 3,     /* symbol missing from a module               */
    RTCG_ERR_COMPILE = 4,       /* NVRTC rejected the source (see log)        */
    RTCG_ERR_NO_DEVICE = 5,     /* libcuda missing or no CUDA device          */
    RTCG_ERR_INVALID = 6,       /* bad argument to this library               */
    RTCG_ERR_LOAD = 7,          /* module image rejected by the driver        */
    RTCG_ERR_NO_COMPILER = 8    /* libnvrtc could not be loaded               */
};

typedef struct rtcg_module_s *rtcg_module_t;     /* CUmodule   */
typedef struct rtcg_function_s *rtcg_function_t; /* CUfunction */
typedef struct rtcg_stream_s *rtcg_stream_t;     /* CUstream; NULL = legacy default */
typedef struct rtcg_event_s *rtcg_event_t;       /* CUevent    */
typedef struct rtcg_graph_s *rtcg_graph_t;       /* CUgraphExec (instantiated) */

typedef struct rtcg_device_info {
    char name[128];
    int cc_major, cc_minor;
    int sm_count;
    int max_threads_per_sm;
    int max_threads_per_block;
    int l2_bytes;
    int driver_version;
    int mem_clock_khz, mem_bus_width;
    uint64_t total_mem;
} rtcg_device_info;

/* --- library / errors -------------------------------------------------- */
int rtcg_abi_version(void);
/* Message for the last failing call on this thread ("" if none). */
const char *rtcg_last_error(void);

/* --- NVRTC compile backend (replaces src/jit.py:446-474) ---------------- */
int rtcg_nvrtc_version(int *major, int *minor);
/* Compile `source` to a cubin.  On success *image / *image_size hold a
 * malloc'd cubin; *log always receives the (possibly empty) malloc'd compiler
 * log.  Release both with rtcg_free_buffer.  Returns RTCG_ERR_COMPILE when
 * NVRTC reports an error. */
int rtcg_compile(const char *source, const char *program_name,
                 const char *const *options, int num_options,
                 void **image, size_t *image_size, char **log);
void rtcg_free_buffer(void *p);

/* --- devices / contexts -------------------------------------------------- */
int rtcg_init(void);
int rtcg_device_count(int *count);
int rtcg_device_info_get(int device, rtcg_device_info *info);
/* "dddd:bb:dd.f" of a visible device (cuDeviceGetPCIBusId): a process-
 * independent identity (ordinals depend on CUDA_VISIBLE_DEVICES), used to
 * decide whether ranks really run on distinct, peer-reachable GPUs. */
int rtcg_device_pci_bus_id(int device, char *buf, int len);
/* Retain the device's primary context (shared with the CUDA runtime / torch)
 * and make it current on the calling thread. */
int rtcg_set_device(int device);
int rtcg_get_device(int *device);
int rtcg_synchronize(void);
int rtcg_mem_get_info(uint64_t *free_bytes, uint64_t *total_bytes);

/* --- modules (replaces src/jit.py:439-443, :557-564) -------------------- */
int rtcg_module_load(const void *image, size_t image_size, rtcg_module_t *module);
int rtcg_module_unload(rtcg_module_t module);
int rtcg_module_function(rtcg_module_t module, const char *name,
                         rtcg_function_t *function);
int rtcg_function_occupancy(rtcg_function_t function, int block_threads,
                            size_t dynamic_smem, int *blocks_per_sm);
int rtcg_function_registers(rtcg_function_t function, int *num_regs);
/* Opt a function in to more than 48 KB of dynamic shared memory. */
int rtcg_function_set_max_dynamic_smem(rtcg_function_t function, int bytes);

/* --- launch (replaces KernelHandle.__call__, src/jit.py:553-554) --------
 * `params` follows cuLaunchKernel: params[k] points at the value of kernel
 * parameter k -- the same "pack of pointers to argument values" convention
 * as the reference's void **args. */
int rtcg_launch(rtcg_function_t function, unsigned grid, unsigned block,
                unsigned dynamic_smem, rtcg_stream_t stream, void **params);

/* rtcg_launch with launch flags.  RTCG_LAUNCH_OVERLAP_PREVIOUS: programmatic
 * dependent launch -- the kernel may start while the previous kernel on the
 * stream drains, up to its first `griddepcontrol.wait`; the caller asserts the
 * previous kernel writes nothing this one reads before that point (the
 * reduction templates wait before touching their scratch). */
#define RTCG_LAUNCH_OVERLAP_PREVIOUS 1u
int rtcg_launch_ex(rtcg_function_t function, unsigned grid, unsigned block,
                   unsigned dynamic_smem, rtcg_stream_t stream, void **params, unsigned flags);

/* --- device memory (replaces src/ndarray.py:158-160, :216, :316-336) ----- */
int rtcg_mem_alloc(uint64_t nbytes, uint64_t *dptr);
int rtcg_mem_free(uint64_t dptr);
/* Stream-ordered allocation from the device's default memory pool (release
 * threshold raised so freed memory stays cached by the driver): allocation
 * and free are ordered with kernels on `stream` and never synchronise. */
int rtcg_mem_alloc_async(uint64_t nbytes, rtcg_stream_t stream, uint64_t *dptr);
int rtcg_mem_free_async(uint64_t dptr, rtcg_stream_t stream);
/* Synchronise the current device and return the unused memory cached by its
 * stream-ordered pool to the driver (used before retrying an allocation that
 * failed with RTCG_ERR_OUT_OF_MEMORY). */
int rtcg_mem_trim(void);
int rtcg_memset_async(uint64_t dptr, unsigned char value, uint64_t nbytes,
                      rtcg_stream_t stream);
int rtcg_memcpy_htod_async(uint64_t dst, const void *src, uint64_t nbytes,
                           rtcg_stream_t stream);
int rtcg_memcpy_dtoh_async(void *dst, uint64_t src, uint64_t nbytes,
                           rtcg_stream_t stream);
int rtcg_memcpy_dtod_async(uint64_t dst, uint64_t src, uint64_t nbytes,
                           rtcg_stream_t stream);
/* Host <-> device copies that pick the fast path for the host buffer:
 * page-locked memory is DMA'd directly (asynchronously); pageable memory is
 * staged through pinned double buffers, the host-side memcpy parallelised
 * over worker threads and overlapped with the DMA of the previous chunk.
 * HtoD returns once `src` may be reused; DtoH returns once `dst` is filled.
 * (NdArray.copy_from_host / to_host, src/ndarray.py:316-336.) */
int rtcg_copy_htod(uint64_t dst, const void *src, uint64_t nbytes, rtcg_stream_t stream);
int rtcg_copy_dtoh(void *dst, uint64_t src, uint64_t nbytes, rtcg_stream_t stream);

/* Page-locked host memory for fast transfers. */
int rtcg_host_alloc(uint64_t nbytes, void **ptr);
int rtcg_host_free(void *ptr);
int rtcg_host_register(void *ptr, uint64_t nbytes);
int rtcg_host_unregister(void *ptr);
/* *pinned = 1 when `ptr` lies in page-locked host memory (allocated or
 * registered), else 0: the test rtcg_copy_htod / rtcg_copy_dtoh use to take
 * the direct DMA path. */
int rtcg_host_is_pinned(const void *ptr, int *pinned);

/* --- streams / events ---------------------------------------------------- */
int rtcg_stream_create(rtcg_stream_t *stream);
int rtcg_stream_destroy(rtcg_stream_t stream);
int rtcg_stream_synchronize(rtcg_stream_t stream);
int rtcg_event_create(rtcg_event_t *event);
int rtcg_event_destroy(rtcg_event_t event);
int rtcg_event_record(rtcg_event_t event, rtcg_stream_t stream);
/* Work submitted to `stream` after this call waits for `event` (cuStreamWaitEvent);
 * streamed host calls order their private streams after the caller's stream. */
int rtcg_stream_wait_event(rtcg_stream_t stream, rtcg_event_t event);
/* *capturing = 1 while `stream` is being captured into a CUDA graph
 * (cuStreamIsCapturing): overlapped reductions fall back to their serial
 * scratch slot there, since a replay re-runs baked launch numbers. */
int rtcg_stream_is_capturing(rtcg_stream_t stream, int *capturing);
int rtcg_event_synchronize(rtcg_event_t event);
int rtcg_event_elapsed_ms(rtcg_event_t start, rtcg_event_t end, float *ms);

/* --- CUDA graphs (no reference equivalent: replays a captured sequence of
 * generated-kernel launches with one launch, for launch-bound small-n
 * chains).  Capture must use a created stream, not the legacy default. */
int rtcg_stream_begin_capture(rtcg_stream_t stream);
/* Ends capture and instantiates the graph. */
int rtcg_stream_end_capture(rtcg_stream_t stream, rtcg_graph_t *graph);
int rtcg_graph_launch(rtcg_graph_t graph, rtcg_stream_t stream);
int rtcg_graph_destroy(rtcg_graph_t graph);

/* --- peer memory (no reference equivalent: the reference's workers share one
 * address space).  The multi-GPU reduction exchanges its per-GPU accumulators
 * inside the reduction kernel itself, with stores into every peer's mailbox
 * over NVLink / NVSwitch (parallel.PeerMailbox; replaces the ordered host fold
 * of worker partials, src/reduction.py:211-216, at GPU granularity).
 * Mailboxes are rtcg_mem_alloc buffers shared across the one-process-per-GPU
 * ranks with CUDA IPC handles (64 opaque bytes). */
int rtcg_ipc_get_handle(uint64_t dptr, unsigned char handle[64]);
/* Maps a peer process's buffer (peer access enabled lazily). */
int rtcg_ipc_open_handle(const unsigned char handle[64], uint64_t *dptr);
int rtcg_ipc_close_handle(uint64_t dptr);
int rtcg_device_can_access_peer(int device, int peer, int *can);

#ifdef __cplusplus
}
#endif

#endif /* RTCG_B200_H */
