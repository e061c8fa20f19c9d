// librtcg_b200.so -- NVRTC + CUDA driver runtime behind the C ABI declared in
// include/rtcg_b200.h.  See that header for which reference seam each entry
// point replaces.
//
// Design notes
//  * libcuda.so.1 and libnvrtc.so.12 are dlopen'd on first use, so the library
//    loads on GPU-less build hosts (where NVRTC still compiles sm_100a cubins).
//  * Contexts: the device's *primary* context is retained and made current, so
//    modules, allocations and streams interoperate with the CUDA runtime (and
//    torch) in the same process.
//  * Errors: every call returns an rtcg_status and stores a message in a
//    thread-local buffer read by rtcg_last_error().

#include "../../include/rtcg_b200.h"

#include <cuda.h>
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

namespace {

thread_local std::string g_error;

int fail(int status, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
    return status;
}

// ---------------------------------------------------------------- driver API

template <class Sig>
using fnptr = Sig *;

struct Driver {
    bool tried = false;
    void *handle = nullptr;
    std::string why;
#define RTCG_DRIVER_FNS(X)                                                     \
    X(cuInit, CUresult(unsigned))                                          \
    X(cuDriverGetVersion, CUresult(int *))                                 \
    X(cuDeviceGetCount, CUresult(int *))                                   \
    X(cuDeviceGet, CUresult(CUdevice *, int))                              \
    X(cuDeviceGetName, CUresult(char *, int, CUdevice))                    \
    X(cuDeviceGetAttribute, CUresult(int *, CUdevice_attribute, CUdevice)) \
    X(cuDeviceTotalMem_v2, CUresult(size_t *, CUdevice))                   \
    X(cuDevicePrimaryCtxRetain, CUresult(CUcontext *, CUdevice))           \
    X(cuCtxSetCurrent, CUresult(CUcontext))                                \
    X(cuCtxGetCurrent, CUresult(CUcontext *))                              \
    X(cuCtxGetDevice, CUresult(CUdevice *))                                \
    X(cuCtxSynchronize, CUresult(void))                                    \
    X(cuMemGetInfo_v2, CUresult(size_t *, size_t *))                       \
    X(cuModuleLoadData, CUresult(CUmodule *, const void *))                \
    X(cuModuleUnload, CUresult(CUmodule))                                  \
    X(cuModuleGetFunction, CUresult(CUfunction *, CUmodule, const char *)) \
    X(cuFuncGetAttribute, CUresult(int *, CUfunction_attribute, CUfunction)) \
    X(cuFuncSetAttribute, CUresult(CUfunction, CUfunction_attribute, int))   \
    X(cuOccupancyMaxActiveBlocksPerMultiprocessor,                             \
      CUresult(int *, CUfunction, int, size_t))                            \
    X(cuLaunchKernel, CUresult(CUfunction, unsigned, unsigned, unsigned,   \
                                   unsigned, unsigned, unsigned, unsigned,     \
                                   CUstream, void **, void **))                \
    X(cuMemAlloc_v2, CUresult(CUdeviceptr *, size_t))                      \
    X(cuMemFree_v2, CUresult(CUdeviceptr))                                 \
    X(cuMemAllocAsync, CUresult(CUdeviceptr *, size_t, CUstream))            \
    X(cuMemFreeAsync, CUresult(CUdeviceptr, CUstream))                       \
    X(cuDeviceGetDefaultMemPool, CUresult(CUmemoryPool *, CUdevice))         \
    X(cuMemPoolSetAttribute, CUresult(CUmemoryPool, CUmemPool_attribute, void *)) \
    X(cuMemPoolTrimTo, CUresult(CUmemoryPool, size_t))                       \
    X(cuMemsetD8Async, CUresult(CUdeviceptr, unsigned char, size_t, CUstream)) \
    X(cuMemcpyHtoDAsync_v2,                                                    \
      CUresult(CUdeviceptr, const void *, size_t, CUstream))               \
    X(cuMemcpyDtoHAsync_v2, CUresult(void *, CUdeviceptr, size_t, CUstream)) \
    X(cuMemcpyDtoDAsync_v2,                                                    \
      CUresult(CUdeviceptr, CUdeviceptr, size_t, CUstream))                \
    X(cuMemHostAlloc, CUresult(void **, size_t, unsigned))                 \
    X(cuMemFreeHost, CUresult(void *))                                     \
    X(cuMemHostRegister_v2, CUresult(void *, size_t, unsigned))            \
    X(cuMemHostUnregister, CUresult(void *))                               \
    X(cuPointerGetAttributes,                                                  \
      CUresult(unsigned, CUpointer_attribute *, void **, CUdeviceptr))     \
    X(cuStreamCreate, CUresult(CUstream *, unsigned))                      \
    X(cuStreamDestroy_v2, CUresult(CUstream))                              \
    X(cuStreamSynchronize, CUresult(CUstream))                             \
    X(cuStreamWaitEvent, CUresult(CUstream, CUevent, unsigned))            \
    X(cuStreamIsCapturing, CUresult(CUstream, CUstreamCaptureStatus *))     \
    X(cuEventCreate, CUresult(CUevent *, unsigned))                        \
    X(cuEventDestroy_v2, CUresult(CUevent))                                \
    X(cuEventRecord, CUresult(CUevent, CUstream))                          \
    X(cuEventSynchronize, CUresult(CUevent))                               \
    X(cuEventElapsedTime, CUresult(float *, CUevent, CUevent))             \
    X(cuGetErrorName, CUresult(CUresult, const char **))                   \
    X(cuStreamBeginCapture_v2, CUresult(CUstream, CUstreamCaptureMode))      \
    X(cuStreamEndCapture, CUresult(CUstream, CUgraph *))                     \
    X(cuGraphInstantiateWithFlags, CUresult(CUgraphExec *, CUgraph, unsigned long long)) \
    X(cuGraphLaunch, CUresult(CUgraphExec, CUstream))                        \
    X(cuGraphExecDestroy, CUresult(CUgraphExec))                             \
    X(cuGraphDestroy, CUresult(CUgraph))                                     \
    X(cuLaunchKernelEx, CUresult(const CUlaunchConfig *, CUfunction, void **, void **)) \
    X(cuIpcGetMemHandle, CUresult(CUipcMemHandle *, CUdeviceptr))            \
    X(cuIpcOpenMemHandle_v2, CUresult(CUdeviceptr *, CUipcMemHandle, unsigned)) \
    X(cuIpcCloseMemHandle, CUresult(CUdeviceptr))                            \
    X(cuDeviceCanAccessPeer, CUresult(int *, CUdevice, CUdevice))            \
    X(cuDeviceGetPCIBusId, CUresult(char *, int, CUdevice))                  \
    X(cuGetErrorString, CUresult(CUresult, const char **))
#define RTCG_DECLARE(name, sig) fnptr<sig> name = nullptr;
    RTCG_DRIVER_FNS(RTCG_DECLARE)
#undef RTCG_DECLARE
    int init_status = RTCG_ERR_NO_DEVICE;
};

Driver g_drv;
std::mutex g_drv_mutex;
std::vector<CUcontext> g_primary;  // per device, retained once
thread_local int t_device = -1;

const char *cu_name(CUresult r) {
    const char *s = nullptr;
    if (g_drv.cuGetErrorName && g_drv.cuGetErrorName(r, &s) == CUDA_SUCCESS && s)
        return s;
    return "CUDA_ERROR_?";
}

const char *cu_text(CUresult r) {
    const char *s = nullptr;
    if (g_drv.cuGetErrorString && g_drv.cuGetErrorString(r, &s) == CUDA_SUCCESS && s)
        return s;
    return "";
}

int cu_fail(CUresult r, const char *what) {
    int status = RTCG_ERR_CUDA;
    if (r == CUDA_ERROR_OUT_OF_MEMORY) status = RTCG_ERR_OUT_OF_MEMORY;
    else if (r == CUDA_ERROR_NOT_FOUND) status = RTCG_ERR_NOT_FOUND;
    else if (r == CUDA_ERROR_INVALID_IMAGE || r == CUDA_ERROR_NO_BINARY_FOR_GPU ||
             r == CUDA_ERROR_INVALID_PTX || r == CUDA_ERROR_UNSUPPORTED_PTX_VERSION)
        status = RTCG_ERR_LOAD;
    else if (r == CUDA_ERROR_NO_DEVICE) status = RTCG_ERR_NO_DEVICE;
    return fail(status, "%s failed: %s (%d) %s", what, cu_name(r), (int)r, cu_text(r));
}

// Load libcuda and cuInit once; later calls return the cached outcome.
int driver_ready() {
    std::lock_guard<std::mutex> lock(g_drv_mutex);
    if (g_drv.tried) {
        if (g_drv.init_status != RTCG_OK) return fail(g_drv.init_status, "%s", g_drv.why.c_str());
        return RTCG_OK;
    }
    g_drv.tried = true;
    g_drv.handle = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!g_drv.handle) {
        g_drv.why = std::string("cannot load libcuda.so.1 (no NVIDIA driver): ") + dlerror();
        return fail(g_drv.init_status, "%s", g_drv.why.c_str());
    }
#define RTCG_RESOLVE(name, sig)                                                    \
    g_drv.name = reinterpret_cast<fnptr<sig>>(dlsym(g_drv.handle, #name));          \
    if (!g_drv.name) {                                                             \
        g_drv.why = "libcuda.so.1 lacks symbol " #name;                            \
        return fail(g_drv.init_status, "%s", g_drv.why.c_str());                   \
    }
    RTCG_DRIVER_FNS(RTCG_RESOLVE)
#undef RTCG_RESOLVE
    CUresult r = g_drv.cuInit(0);
    if (r != CUDA_SUCCESS) {
        g_drv.why = std::string("cuInit failed: ") + cu_name(r) + " " + cu_text(r);
        return fail(g_drv.init_status, "%s", g_drv.why.c_str());
    }
    int count = 0;
    if (g_drv.cuDeviceGetCount(&count) != CUDA_SUCCESS || count == 0) {
        g_drv.why = "no CUDA device visible";
        return fail(g_drv.init_status, "%s", g_drv.why.c_str());
    }
    g_primary.assign(count, nullptr);
    g_drv.init_status = RTCG_OK;
    return RTCG_OK;
}

// Make sure the calling thread has a current context (device 0 by default,
// or the device torch / the caller already made current).
int ensure_context() {
    int s = driver_ready();
    if (s != RTCG_OK) return s;
    if (t_device >= 0) return RTCG_OK;
    CUcontext cur = nullptr;
    if (g_drv.cuCtxGetCurrent(&cur) == CUDA_SUCCESS && cur) {
        CUdevice dev;
        if (g_drv.cuCtxGetDevice(&dev) == CUDA_SUCCESS) {
            t_device = (int)dev;
            return RTCG_OK;
        }
    }
    return rtcg_set_device(0);
}

#define CU_CALL(expr, what)                          \
    do {                                             \
        CUresult r_ = (expr);                        \
        if (r_ != CUDA_SUCCESS) return cu_fail(r_, what); \
    } while (0)

#define NEED_CONTEXT()                      \
    do {                                    \
        int s_ = ensure_context();          \
        if (s_ != RTCG_OK) return s_;       \
    } while (0)

// ---------------------------------------------------------------- NVRTC

typedef int nvrtcResult_t;
struct Nvrtc {
    bool tried = false;
    void *handle = nullptr;
    std::string why;
    nvrtcResult_t (*nvrtcVersion)(int *, int *) = nullptr;
    nvrtcResult_t (*nvrtcCreateProgram)(void **, const char *, const char *, int,
                                        const char *const *, const char *const *) = nullptr;
    nvrtcResult_t (*nvrtcDestroyProgram)(void **) = nullptr;
    nvrtcResult_t (*nvrtcCompileProgram)(void *, int, const char *const *) = nullptr;
    nvrtcResult_t (*nvrtcGetCUBINSize)(void *, size_t *) = nullptr;
    nvrtcResult_t (*nvrtcGetCUBIN)(void *, char *) = nullptr;
    nvrtcResult_t (*nvrtcGetProgramLogSize)(void *, size_t *) = nullptr;
    nvrtcResult_t (*nvrtcGetProgramLog)(void *, char *) = nullptr;
    const char *(*nvrtcGetErrorString)(nvrtcResult_t) = nullptr;
};

Nvrtc g_nvrtc;
std::mutex g_nvrtc_mutex;

int nvrtc_ready() {
    std::lock_guard<std::mutex> lock(g_nvrtc_mutex);
    if (g_nvrtc.tried) {
        if (!g_nvrtc.handle) return fail(RTCG_ERR_NO_COMPILER, "%s", g_nvrtc.why.c_str());
        return RTCG_OK;
    }
    g_nvrtc.tried = true;
    const char *env = getenv("RTCG_NVRTC_LIBRARY");
    const char *candidates[] = {env, "libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12",
                                "libnvrtc.so"};
    for (const char *c : candidates) {
        if (!c || !*c) continue;
        g_nvrtc.handle = dlopen(c, RTLD_NOW | RTLD_LOCAL);
        if (g_nvrtc.handle) break;
    }
    if (!g_nvrtc.handle) {
        g_nvrtc.why = std::string("cannot load libnvrtc.so.12: ") + dlerror();
        return fail(RTCG_ERR_NO_COMPILER, "%s", g_nvrtc.why.c_str());
    }
#define RTCG_NV(name)                                                             \
    *reinterpret_cast<void **>(&g_nvrtc.name) = dlsym(g_nvrtc.handle, #name);     \
    if (!g_nvrtc.name) {                                                          \
        g_nvrtc.why = "libnvrtc lacks symbol " #name;                             \
        dlclose(g_nvrtc.handle);                                                  \
        g_nvrtc.handle = nullptr;                                                 \
        return fail(RTCG_ERR_NO_COMPILER, "%s", g_nvrtc.why.c_str());             \
    }
    RTCG_NV(nvrtcVersion)
    RTCG_NV(nvrtcCreateProgram)
    RTCG_NV(nvrtcDestroyProgram)
    RTCG_NV(nvrtcCompileProgram)
    RTCG_NV(nvrtcGetCUBINSize)
    RTCG_NV(nvrtcGetCUBIN)
    RTCG_NV(nvrtcGetProgramLogSize)
    RTCG_NV(nvrtcGetProgramLog)
    RTCG_NV(nvrtcGetErrorString)
#undef RTCG_NV
    return RTCG_OK;
}

char *dup_string(const std::string &s) {
    char *p = static_cast<char *>(malloc(s.size() + 1));
    if (p) memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

}  // namespace

// ============================================================== public ABI

extern "C" {

int rtcg_abi_version(void) { return RTCG_ABI_VERSION; }

const char *rtcg_last_error(void) { return g_error.c_str(); }

void rtcg_free_buffer(void *p) { free(p); }

int rtcg_nvrtc_version(int *major, int *minor) {
    int s = nvrtc_ready();
    if (s != RTCG_OK) return s;
    if (g_nvrtc.nvrtcVersion(major, minor) != 0) return fail(RTCG_ERR_NO_COMPILER, "nvrtcVersion failed");
    return RTCG_OK;
}

int rtcg_compile(const char *source, const char *program_name, const char *const *options,
                 int num_options, void **image, size_t *image_size, char **log) {
    if (image) *image = nullptr;
    if (image_size) *image_size = 0;
    if (log) *log = nullptr;
    if (!source || !image || !image_size || num_options < 0)
        return fail(RTCG_ERR_INVALID, "rtcg_compile: null argument");
    int s = nvrtc_ready();
    if (s != RTCG_OK) return s;
    void *prog = nullptr;
    int r = g_nvrtc.nvrtcCreateProgram(&prog, source, program_name ? program_name : "rtcg.cu",
                                       0, nullptr, nullptr);
    if (r != 0)
        return fail(RTCG_ERR_COMPILE, "nvrtcCreateProgram: %s", g_nvrtc.nvrtcGetErrorString(r));
    int cr = g_nvrtc.nvrtcCompileProgram(prog, num_options, options);
    size_t log_size = 0;
    std::string text;
    if (g_nvrtc.nvrtcGetProgramLogSize(prog, &log_size) == 0 && log_size > 1) {
        text.resize(log_size);
        g_nvrtc.nvrtcGetProgramLog(prog, &text[0]);
        text.resize(strlen(text.c_str()));
    }
    if (log) *log = dup_string(text);
    if (cr != 0) {
        g_nvrtc.nvrtcDestroyProgram(&prog);
        return fail(RTCG_ERR_COMPILE, "nvrtcCompileProgram: %s", g_nvrtc.nvrtcGetErrorString(cr));
    }
    size_t n = 0;
    if (g_nvrtc.nvrtcGetCUBINSize(prog, &n) != 0 || n == 0) {
        g_nvrtc.nvrtcDestroyProgram(&prog);
        return fail(RTCG_ERR_COMPILE,
                    "NVRTC produced no cubin (is -arch=sm_XXX a real architecture?)");
    }
    char *buf = static_cast<char *>(malloc(n));
    if (!buf) {
        g_nvrtc.nvrtcDestroyProgram(&prog);
        return fail(RTCG_ERR_OUT_OF_MEMORY, "host malloc(%zu) failed", n);
    }
    g_nvrtc.nvrtcGetCUBIN(prog, buf);
    g_nvrtc.nvrtcDestroyProgram(&prog);
    *image = buf;
    *image_size = n;
    return RTCG_OK;
}

int rtcg_init(void) { return driver_ready(); }

int rtcg_device_count(int *count) {
    int s = driver_ready();
    if (s != RTCG_OK) return s;
    CU_CALL(g_drv.cuDeviceGetCount(count), "cuDeviceGetCount");
    return RTCG_OK;
}

int rtcg_device_info_get(int device, rtcg_device_info *info) {
    int s = driver_ready();
    if (s != RTCG_OK) return s;
    if (!info) return fail(RTCG_ERR_INVALID, "null info");
    memset(info, 0, sizeof *info);
    CUdevice dev;
    CU_CALL(g_drv.cuDeviceGet(&dev, device), "cuDeviceGet");
    CU_CALL(g_drv.cuDeviceGetName(info->name, sizeof info->name - 1, dev), "cuDeviceGetName");
    struct { int *dst; CUdevice_attribute a; } attrs[] = {
        {&info->cc_major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR},
        {&info->cc_minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR},
        {&info->sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT},
        {&info->max_threads_per_sm, CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_MULTIPROCESSOR},
        {&info->max_threads_per_block, CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_BLOCK},
        {&info->l2_bytes, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE},
        {&info->mem_clock_khz, CU_DEVICE_ATTRIBUTE_MEMORY_CLOCK_RATE},
        {&info->mem_bus_width, CU_DEVICE_ATTRIBUTE_GLOBAL_MEMORY_BUS_WIDTH},
    };
    for (auto &a : attrs) CU_CALL(g_drv.cuDeviceGetAttribute(a.dst, a.a, dev), "cuDeviceGetAttribute");
    size_t total = 0;
    CU_CALL(g_drv.cuDeviceTotalMem_v2(&total, dev), "cuDeviceTotalMem");
    info->total_mem = total;
    CU_CALL(g_drv.cuDriverGetVersion(&info->driver_version), "cuDriverGetVersion");
    return RTCG_OK;
}

int rtcg_device_pci_bus_id(int device, char *buf, int len) {
    int s = driver_ready();
    if (s != RTCG_OK) return s;
    if (!buf || len < 13) return fail(RTCG_ERR_INVALID, "bus id buffer needs >= 13 bytes");
    CUdevice dev;
    CU_CALL(g_drv.cuDeviceGet(&dev, device), "cuDeviceGet");
    CU_CALL(g_drv.cuDeviceGetPCIBusId(buf, len, dev), "cuDeviceGetPCIBusId");
    return RTCG_OK;
}

int rtcg_set_device(int device) {
    int s = driver_ready();
    if (s != RTCG_OK) return s;
    if (device < 0 || device >= (int)g_primary.size())
        return fail(RTCG_ERR_INVALID, "device %d out of range [0, %zu)", device, g_primary.size());
    CUcontext ctx;
    {
        std::lock_guard<std::mutex> lock(g_drv_mutex);
        if (!g_primary[device]) {
            CUdevice dev;
            CU_CALL(g_drv.cuDeviceGet(&dev, device), "cuDeviceGet");
            CU_CALL(g_drv.cuDevicePrimaryCtxRetain(&g_primary[device], dev),
                    "cuDevicePrimaryCtxRetain");
        }
        ctx = g_primary[device];
    }
    CU_CALL(g_drv.cuCtxSetCurrent(ctx), "cuCtxSetCurrent");
    t_device = device;
    return RTCG_OK;
}

int rtcg_get_device(int *device) {
    NEED_CONTEXT();
    *device = t_device;
    return RTCG_OK;
}

int rtcg_synchronize(void) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuCtxSynchronize(), "cuCtxSynchronize");
    return RTCG_OK;
}

int rtcg_mem_get_info(uint64_t *free_bytes, uint64_t *total_bytes) {
    NEED_CONTEXT();
    size_t f = 0, t = 0;
    CU_CALL(g_drv.cuMemGetInfo_v2(&f, &t), "cuMemGetInfo");
    *free_bytes = f;
    *total_bytes = t;
    return RTCG_OK;
}

int rtcg_module_load(const void *image, size_t image_size, rtcg_module_t *module) {
    if (!image || !module || image_size < 4)
        return fail(RTCG_ERR_INVALID, "rtcg_module_load: empty image");
    NEED_CONTEXT();
    CUmodule m;
    CU_CALL(g_drv.cuModuleLoadData(&m, image), "cuModuleLoadData");
    *module = reinterpret_cast<rtcg_module_t>(m);
    return RTCG_OK;
}

int rtcg_module_unload(rtcg_module_t module) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuModuleUnload(reinterpret_cast<CUmodule>(module)), "cuModuleUnload");
    return RTCG_OK;
}

int rtcg_module_function(rtcg_module_t module, const char *name, rtcg_function_t *function) {
    NEED_CONTEXT();
    CUfunction f;
    CUresult r = g_drv.cuModuleGetFunction(&f, reinterpret_cast<CUmodule>(module), name);
    if (r == CUDA_ERROR_NOT_FOUND) return fail(RTCG_ERR_NOT_FOUND, "kernel symbol '%s' not found", name);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuModuleGetFunction");
    // Load the kernel's code now rather than at its first launch (CUDA's lazy
    // loading): a load may wait for running kernels, which must not happen
    // between the launches of kernels that wait on each other (the peer
    // exchange of multi-GPU reductions).  cuFuncLoad is optional (CUDA 12.4+).
    using func_load_t = CUresult (*)(CUfunction);
    static func_load_t func_load =
        reinterpret_cast<func_load_t>(dlsym(g_drv.handle, "cuFuncLoad"));
    if (func_load) {
        r = func_load(f);
        if (r != CUDA_SUCCESS) return cu_fail(r, "cuFuncLoad");
    }
    *function = reinterpret_cast<rtcg_function_t>(f);
    return RTCG_OK;
}

int rtcg_function_occupancy(rtcg_function_t function, int block_threads, size_t dynamic_smem,
                            int *blocks_per_sm) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuOccupancyMaxActiveBlocksPerMultiprocessor(
                blocks_per_sm, reinterpret_cast<CUfunction>(function), block_threads, dynamic_smem),
            "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    return RTCG_OK;
}

int rtcg_function_registers(rtcg_function_t function, int *num_regs) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuFuncGetAttribute(num_regs, CU_FUNC_ATTRIBUTE_NUM_REGS,
                                     reinterpret_cast<CUfunction>(function)),
            "cuFuncGetAttribute");
    return RTCG_OK;
}

int rtcg_function_set_max_dynamic_smem(rtcg_function_t function, int bytes) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuFuncSetAttribute(reinterpret_cast<CUfunction>(function),
                                     CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes),
            "cuFuncSetAttribute(MAX_DYNAMIC_SHARED_SIZE_BYTES)");
    return RTCG_OK;
}

int rtcg_launch(rtcg_function_t function, unsigned grid, unsigned block, unsigned dynamic_smem,
                rtcg_stream_t stream, void **params) {
    if (!function || grid == 0 || block == 0)
        return fail(RTCG_ERR_INVALID, "rtcg_launch: grid=%u block=%u", grid, block);
    NEED_CONTEXT();
    CU_CALL(g_drv.cuLaunchKernel(reinterpret_cast<CUfunction>(function), grid, 1, 1, block, 1, 1,
                                 dynamic_smem, reinterpret_cast<CUstream>(stream), params, nullptr),
            "cuLaunchKernel");
    return RTCG_OK;
}

int rtcg_launch_ex(rtcg_function_t function, unsigned grid, unsigned block,
                   unsigned dynamic_smem, rtcg_stream_t stream, void **params, unsigned flags) {
    if (!(flags & RTCG_LAUNCH_OVERLAP_PREVIOUS))
        return rtcg_launch(function, grid, block, dynamic_smem, stream, params);
    if (!function || grid == 0 || block == 0)
        return fail(RTCG_ERR_INVALID, "rtcg_launch_ex: grid=%u block=%u", grid, block);
    NEED_CONTEXT();
    CUlaunchAttribute attr;
    memset(&attr, 0, sizeof(attr));
    attr.id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr.value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDimX = grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = block;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = dynamic_smem;
    cfg.hStream = reinterpret_cast<CUstream>(stream);
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    CU_CALL(g_drv.cuLaunchKernelEx(&cfg, reinterpret_cast<CUfunction>(function), params, nullptr),
            "cuLaunchKernelEx");
    return RTCG_OK;
}

int rtcg_mem_alloc(uint64_t nbytes, uint64_t *dptr) {
    NEED_CONTEXT();
    CUdeviceptr p = 0;
    CU_CALL(g_drv.cuMemAlloc_v2(&p, nbytes), "cuMemAlloc");
    *dptr = p;
    return RTCG_OK;
}

int rtcg_mem_free(uint64_t dptr) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemFree_v2(dptr), "cuMemFree");
    return RTCG_OK;
}

static std::vector<char> g_pool_ready;  // per device: release threshold raised

int rtcg_mem_alloc_async(uint64_t nbytes, rtcg_stream_t stream, uint64_t *dptr) {
    NEED_CONTEXT();
    {
        std::lock_guard<std::mutex> lock(g_drv_mutex);
        if (g_pool_ready.size() < g_primary.size()) g_pool_ready.assign(g_primary.size(), 0);
        if (!g_pool_ready[t_device]) {
            CUmemoryPool pool;
            CUdevice dev;
            CU_CALL(g_drv.cuDeviceGet(&dev, t_device), "cuDeviceGet");
            CU_CALL(g_drv.cuDeviceGetDefaultMemPool(&pool, dev), "cuDeviceGetDefaultMemPool");
            cuuint64_t keep = ~0ull;
            CU_CALL(g_drv.cuMemPoolSetAttribute(pool, CU_MEMPOOL_ATTR_RELEASE_THRESHOLD, &keep),
                    "cuMemPoolSetAttribute(RELEASE_THRESHOLD)");
            g_pool_ready[t_device] = 1;
        }
    }
    CUdeviceptr p = 0;
    CU_CALL(g_drv.cuMemAllocAsync(&p, nbytes, reinterpret_cast<CUstream>(stream)),
            "cuMemAllocAsync");
    *dptr = p;
    return RTCG_OK;
}

int rtcg_mem_trim(void) {
    NEED_CONTEXT();
    CUdevice dev;
    CUmemoryPool pool;
    CU_CALL(g_drv.cuCtxSynchronize(), "cuCtxSynchronize");
    CU_CALL(g_drv.cuDeviceGet(&dev, t_device), "cuDeviceGet");
    CU_CALL(g_drv.cuDeviceGetDefaultMemPool(&pool, dev), "cuDeviceGetDefaultMemPool");
    CU_CALL(g_drv.cuMemPoolTrimTo(pool, 0), "cuMemPoolTrimTo");
    return RTCG_OK;
}

int rtcg_mem_free_async(uint64_t dptr, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemFreeAsync(dptr, reinterpret_cast<CUstream>(stream)), "cuMemFreeAsync");
    return RTCG_OK;
}

int rtcg_memset_async(uint64_t dptr, unsigned char value, uint64_t nbytes, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemsetD8Async(dptr, value, nbytes, reinterpret_cast<CUstream>(stream)),
            "cuMemsetD8Async");
    return RTCG_OK;
}

int rtcg_memcpy_htod_async(uint64_t dst, const void *src, uint64_t nbytes, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemcpyHtoDAsync_v2(dst, src, nbytes, reinterpret_cast<CUstream>(stream)),
            "cuMemcpyHtoDAsync");
    return RTCG_OK;
}

int rtcg_memcpy_dtoh_async(void *dst, uint64_t src, uint64_t nbytes, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemcpyDtoHAsync_v2(dst, src, nbytes, reinterpret_cast<CUstream>(stream)),
            "cuMemcpyDtoHAsync");
    return RTCG_OK;
}

int rtcg_memcpy_dtod_async(uint64_t dst, uint64_t src, uint64_t nbytes, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemcpyDtoDAsync_v2(dst, src, nbytes, reinterpret_cast<CUstream>(stream)),
            "cuMemcpyDtoDAsync");
    return RTCG_OK;
}

// ---------------------------------------------------------------- staged copies
//
// Pageable host memory cannot be DMA'd; the driver stages it through a small
// bounce buffer with one thread (~11 GB/s HtoD on the B200 box).  The copy
// engine instead splits a transfer into one contiguous slice per worker
// thread; every worker owns two pinned lane buffers and pipelines
//   HtoD: host memcpy (non-temporal stores) into lane buffer -> async DMA
//   DtoH: async DMA into lane buffer -> host memcpy out of it
// on the caller's stream, so host-side copying (the bound: host DRAM) runs on
// many cores while the DMA engine stays busy.  One engine per device, created
// on first use, workers persistent; calls are serialised per engine.

namespace {

constexpr size_t kLaneBytes = 4u << 20;     // per lane buffer (2 per worker)
constexpr size_t kDirectBelow = 1u << 20;   // small copies: let the driver stage

// 64-byte blocks of 16-byte non-temporal stores: no read-for-ownership of
// the destination, which would otherwise add a third pass over host DRAM
void stream_copy(void *dst, const void *src, size_t n) {
#if defined(__x86_64__)
    static const bool nt = [] {
        const char *env = getenv("RTCG_COPY_NT");
        return !(env && env[0] == '0');
    }();
    char *d = static_cast<char *>(dst);
    const char *s = static_cast<const char *>(src);
    if (!nt || n < 4096) {
        memcpy(d, s, n);
        return;
    }
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
    memcpy(d, s, head);
    d += head, s += head, n -= head;
    const size_t body = n & ~size_t(63);
    for (size_t i = 0; i < body; i += 64) {
        __m128i x0 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i));
        __m128i x1 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 16));
        __m128i x2 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 32));
        __m128i x3 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i *>(d + i), x0);
        _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 16), x1);
        _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 32), x2);
        _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 48), x3);
    }
    _mm_sfence();
    memcpy(d + body, s + body, n - body);
#else
    memcpy(dst, src, n);
#endif
}

// Page-locked (cuMemHostAlloc'd or registered) host memory reports
// CU_MEMORYTYPE_HOST; ordinary pageable memory is not a CUDA pointer, for
// which cuPointerGetAttributes (unlike cuMemHostGetFlags) returns success
// with a zero type instead of an API error.
bool is_pinned(const void *p) {
    CUpointer_attribute attr = CU_POINTER_ATTRIBUTE_MEMORY_TYPE;
    unsigned type = 0;
    void *data = &type;
    return g_drv.cuPointerGetAttributes(1, &attr, &data, reinterpret_cast<CUdeviceptr>(p)) ==
               CUDA_SUCCESS &&
           type == CU_MEMORYTYPE_HOST;
}

struct CopyJob {
    bool to_device = true;
    uint64_t dev = 0;
    char *host = nullptr;
    uint64_t nbytes = 0;
    size_t slice = 0;
    CUstream stream = nullptr;
};

struct Lane {
    void *buf[2] = {};
    CUevent done[2] = {};
    CUresult err = CUDA_SUCCESS;
    const char *what = "";
};

class CopyEngine {
  public:
    CopyEngine(CUcontext ctx, unsigned workers) : ctx_(ctx), lanes_(workers), pid_(getpid()) {}

    int start() {
        for (auto &lane : lanes_)
            for (int b = 0; b < 2; ++b) {
                CU_CALL(g_drv.cuMemHostAlloc(&lane.buf[b], kLaneBytes, CU_MEMHOSTALLOC_PORTABLE),
                        "cuMemHostAlloc(copy lane)");
                CU_CALL(g_drv.cuEventCreate(&lane.done[b], CU_EVENT_DISABLE_TIMING),
                        "cuEventCreate(copy lane)");
            }
        for (unsigned w = 1; w < lanes_.size(); ++w)
            std::thread([this, w] { worker(w); }).detach();  // engine lives for the process
        return RTCG_OK;
    }

    bool forked() const { return getpid() != pid_; }

    int run(const CopyJob &job) {
        std::lock_guard<std::mutex> call(call_mutex_);
        const unsigned active = (unsigned)std::min<uint64_t>(
            lanes_.size(), (job.nbytes + kLaneBytes - 1) / kLaneBytes);
        {
            std::lock_guard<std::mutex> lock(m_);
            job_ = job;
            job_.slice = ((job.nbytes + active - 1) / active + 63) & ~size_t(63);
            active_ = active;
            pending_ = active - 1;
            ++generation_;
        }
        wake_.notify_all();
        run_lane(0);
        std::unique_lock<std::mutex> lock(m_);
        done_.wait(lock, [this] { return pending_ == 0; });
        for (unsigned w = 0; w < active; ++w)
            if (lanes_[w].err != CUDA_SUCCESS) return cu_fail(lanes_[w].err, lanes_[w].what);
        return RTCG_OK;
    }

  private:
    void worker(unsigned w) {
        g_drv.cuCtxSetCurrent(ctx_);
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lock(m_);
                wake_.wait(lock, [&] { return generation_ != seen; });
                seen = generation_;
                if (w >= active_) continue;
            }
            run_lane(w);
            std::lock_guard<std::mutex> lock(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }

#define LANE_CALL(expr, name)                  \
    do {                                       \
        CUresult r_ = (expr);                  \
        if (r_ != CUDA_SUCCESS) {              \
            lane.err = r_, lane.what = name;   \
            return;                            \
        }                                      \
    } while (0)

    void run_lane(unsigned w) {
        Lane &lane = lanes_[w];
        lane.err = CUDA_SUCCESS;
        const CopyJob &job = job_;
        const uint64_t lo = std::min<uint64_t>(job.nbytes, w * job.slice);
        const uint64_t hi = std::min<uint64_t>(job.nbytes, lo + job.slice);
        const uint64_t chunks = (hi - lo + kLaneBytes - 1) / kLaneBytes;
        auto len = [&](uint64_t k) { return (size_t)std::min<uint64_t>(kLaneBytes, hi - lo - k * kLaneBytes); };
        if (job.to_device) {
            for (uint64_t k = 0; k < chunks; ++k) {
                const int b = k & 1;
                const uint64_t off = lo + k * kLaneBytes;
                LANE_CALL(g_drv.cuEventSynchronize(lane.done[b]), "cuEventSynchronize(copy lane)");
                stream_copy(lane.buf[b], job.host + off, len(k));
                LANE_CALL(g_drv.cuMemcpyHtoDAsync_v2(job.dev + off, lane.buf[b], len(k), job.stream),
                          "cuMemcpyHtoDAsync(staged)");
                LANE_CALL(g_drv.cuEventRecord(lane.done[b], job.stream), "cuEventRecord(copy lane)");
            }
            return;  // the host slice is no longer referenced; DMA may be in flight
        }
        auto issue = [&](uint64_t k) -> CUresult {
            const int b = k & 1;
            CUresult r = g_drv.cuEventSynchronize(lane.done[b]);  // earlier user of buf[b]
            if (r == CUDA_SUCCESS)
                r = g_drv.cuMemcpyDtoHAsync_v2(lane.buf[b], job.dev + lo + k * kLaneBytes, len(k),
                                               job.stream);
            if (r == CUDA_SUCCESS) r = g_drv.cuEventRecord(lane.done[b], job.stream);
            return r;
        };
        if (chunks) LANE_CALL(issue(0), "cuMemcpyDtoHAsync(staged)");
        for (uint64_t k = 0; k < chunks; ++k) {
            if (k + 1 < chunks) LANE_CALL(issue(k + 1), "cuMemcpyDtoHAsync(staged)");
            const int b = k & 1;
            LANE_CALL(g_drv.cuEventSynchronize(lane.done[b]), "cuEventSynchronize(copy lane)");
            stream_copy(job.host + lo + k * kLaneBytes, lane.buf[b], len(k));
        }
    }
#undef LANE_CALL

    CUcontext ctx_;
    std::vector<Lane> lanes_;
    pid_t pid_;
    std::mutex call_mutex_, m_;
    std::condition_variable wake_, done_;
    CopyJob job_;
    uint64_t generation_ = 0;
    unsigned active_ = 0, pending_ = 0;
};

std::mutex g_engine_mutex;
std::vector<CopyEngine *> g_engines;  // per device, leaked at exit on purpose

int copy_engine(CopyEngine *&out) {
    std::lock_guard<std::mutex> lock(g_engine_mutex);
    if ((int)g_engines.size() <= t_device) g_engines.resize(t_device + 1, nullptr);
    CopyEngine *&e = g_engines[t_device];
    if (!e || e->forked()) {  // a forked child has none of the parent's workers
        CUcontext ctx = nullptr;
        CU_CALL(g_drv.cuCtxGetCurrent(&ctx), "cuCtxGetCurrent");
        static const unsigned workers = [] {
            const char *env = getenv("RTCG_COPY_THREADS");  // probing knob
            unsigned hw = std::max(1u, std::thread::hardware_concurrency());
            return env && atoi(env) > 0 ? (unsigned)atoi(env) : std::min(hw, 8u);  // 8: measured best
        }();
        auto *fresh = new CopyEngine(ctx, workers);
        int st = fresh->start();
        if (st != RTCG_OK) return st;  // partially set up engine leaks; rare
        e = fresh;
    }
    out = e;
    return RTCG_OK;
}

}  // namespace

int rtcg_copy_htod(uint64_t dst, const void *src, uint64_t nbytes, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CUstream s = reinterpret_cast<CUstream>(stream);
    if (nbytes < kDirectBelow || is_pinned(src)) {
        CU_CALL(g_drv.cuMemcpyHtoDAsync_v2(dst, src, nbytes, s), "cuMemcpyHtoDAsync");
        return RTCG_OK;
    }
    CopyEngine *e = nullptr;
    int st = copy_engine(e);
    if (st != RTCG_OK) return st;
    CopyJob job;
    job.to_device = true, job.dev = dst, job.host = const_cast<char *>(static_cast<const char *>(src));
    job.nbytes = nbytes, job.stream = s;
    return e->run(job);
}

int rtcg_copy_dtoh(void *dst, uint64_t src, uint64_t nbytes, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CUstream s = reinterpret_cast<CUstream>(stream);
    if (nbytes < kDirectBelow || is_pinned(dst)) {
        CU_CALL(g_drv.cuMemcpyDtoHAsync_v2(dst, src, nbytes, s), "cuMemcpyDtoHAsync");
        CU_CALL(g_drv.cuStreamSynchronize(s), "cuStreamSynchronize");
        return RTCG_OK;
    }
    CopyEngine *e = nullptr;
    int st = copy_engine(e);
    if (st != RTCG_OK) return st;
    CopyJob job;
    job.to_device = false, job.dev = src, job.host = static_cast<char *>(dst);
    job.nbytes = nbytes, job.stream = s;
    return e->run(job);
}

int rtcg_host_alloc(uint64_t nbytes, void **ptr) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemHostAlloc(ptr, nbytes, CU_MEMHOSTALLOC_PORTABLE), "cuMemHostAlloc");
    return RTCG_OK;
}

int rtcg_host_free(void *ptr) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemFreeHost(ptr), "cuMemFreeHost");
    return RTCG_OK;
}

int rtcg_host_register(void *ptr, uint64_t nbytes) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemHostRegister_v2(ptr, nbytes, CU_MEMHOSTREGISTER_PORTABLE),
            "cuMemHostRegister");
    return RTCG_OK;
}

int rtcg_host_unregister(void *ptr) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuMemHostUnregister(ptr), "cuMemHostUnregister");
    return RTCG_OK;
}

int rtcg_host_is_pinned(const void *ptr, int *pinned) {
    if (!pinned) return fail(RTCG_ERR_INVALID, "null output");
    NEED_CONTEXT();
    *pinned = is_pinned(ptr) ? 1 : 0;
    return RTCG_OK;
}

int rtcg_stream_create(rtcg_stream_t *stream) {
    NEED_CONTEXT();
    CUstream s;
    CU_CALL(g_drv.cuStreamCreate(&s, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    *stream = reinterpret_cast<rtcg_stream_t>(s);
    return RTCG_OK;
}

int rtcg_stream_destroy(rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuStreamDestroy_v2(reinterpret_cast<CUstream>(stream)), "cuStreamDestroy");
    return RTCG_OK;
}

int rtcg_stream_synchronize(rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuStreamSynchronize(reinterpret_cast<CUstream>(stream)), "cuStreamSynchronize");
    return RTCG_OK;
}

int rtcg_event_create(rtcg_event_t *event) {
    NEED_CONTEXT();
    CUevent e;
    CU_CALL(g_drv.cuEventCreate(&e, CU_EVENT_DEFAULT), "cuEventCreate");
    *event = reinterpret_cast<rtcg_event_t>(e);
    return RTCG_OK;
}

int rtcg_event_destroy(rtcg_event_t event) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuEventDestroy_v2(reinterpret_cast<CUevent>(event)), "cuEventDestroy");
    return RTCG_OK;
}

int rtcg_event_record(rtcg_event_t event, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuEventRecord(reinterpret_cast<CUevent>(event), reinterpret_cast<CUstream>(stream)),
            "cuEventRecord");
    return RTCG_OK;
}

int rtcg_stream_wait_event(rtcg_stream_t stream, rtcg_event_t event) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuStreamWaitEvent(reinterpret_cast<CUstream>(stream),
                                    reinterpret_cast<CUevent>(event), 0),
            "cuStreamWaitEvent");
    return RTCG_OK;
}

int rtcg_stream_is_capturing(rtcg_stream_t stream, int *capturing) {
    NEED_CONTEXT();
    if (!capturing) return fail(RTCG_ERR_INVALID, "null capturing");
    CUstreamCaptureStatus st = CU_STREAM_CAPTURE_STATUS_NONE;
    CU_CALL(g_drv.cuStreamIsCapturing(reinterpret_cast<CUstream>(stream), &st),
            "cuStreamIsCapturing");
    *capturing = st != CU_STREAM_CAPTURE_STATUS_NONE;
    return RTCG_OK;
}

int rtcg_event_synchronize(rtcg_event_t event) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuEventSynchronize(reinterpret_cast<CUevent>(event)), "cuEventSynchronize");
    return RTCG_OK;
}

int rtcg_event_elapsed_ms(rtcg_event_t start, rtcg_event_t end, float *ms) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuEventElapsedTime(ms, reinterpret_cast<CUevent>(start),
                                     reinterpret_cast<CUevent>(end)),
            "cuEventElapsedTime");
    return RTCG_OK;
}

int rtcg_stream_begin_capture(rtcg_stream_t stream) {
    if (!stream) return fail(RTCG_ERR_INVALID, "cannot capture the legacy default stream");
    NEED_CONTEXT();
    CU_CALL(g_drv.cuStreamBeginCapture_v2(reinterpret_cast<CUstream>(stream),
                                          CU_STREAM_CAPTURE_MODE_RELAXED),
            "cuStreamBeginCapture");
    return RTCG_OK;
}

int rtcg_stream_end_capture(rtcg_stream_t stream, rtcg_graph_t *graph) {
    NEED_CONTEXT();
    CUgraph g = nullptr;
    CU_CALL(g_drv.cuStreamEndCapture(reinterpret_cast<CUstream>(stream), &g),
            "cuStreamEndCapture");
    CUgraphExec exec = nullptr;
    CUresult r = g_drv.cuGraphInstantiateWithFlags(&exec, g, 0);
    g_drv.cuGraphDestroy(g);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuGraphInstantiate");
    *graph = reinterpret_cast<rtcg_graph_t>(exec);
    return RTCG_OK;
}

int rtcg_graph_launch(rtcg_graph_t graph, rtcg_stream_t stream) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuGraphLaunch(reinterpret_cast<CUgraphExec>(graph),
                                reinterpret_cast<CUstream>(stream)),
            "cuGraphLaunch");
    return RTCG_OK;
}

int rtcg_graph_destroy(rtcg_graph_t graph) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuGraphExecDestroy(reinterpret_cast<CUgraphExec>(graph)),
            "cuGraphExecDestroy");
    return RTCG_OK;
}

}  // extern "C"

/* --- peer memory over NVLink / NVSwitch (CUDA IPC) ------------------------ */

int rtcg_ipc_get_handle(uint64_t dptr, unsigned char handle[64]) {
    NEED_CONTEXT();
    if (!handle) return fail(RTCG_ERR_INVALID, "rtcg_ipc_get_handle: null handle");
    CUipcMemHandle h;
    CU_CALL(g_drv.cuIpcGetMemHandle(&h, dptr), "cuIpcGetMemHandle");
    static_assert(sizeof(h.reserved) == 64, "CUipcMemHandle is 64 bytes");
    memcpy(handle, h.reserved, 64);
    return RTCG_OK;
}

int rtcg_ipc_open_handle(const unsigned char handle[64], uint64_t *dptr) {
    NEED_CONTEXT();
    if (!handle || !dptr) return fail(RTCG_ERR_INVALID, "rtcg_ipc_open_handle: null argument");
    CUipcMemHandle h;
    memcpy(h.reserved, handle, 64);
    CUdeviceptr p = 0;
    CU_CALL(g_drv.cuIpcOpenMemHandle_v2(&p, h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS),
            "cuIpcOpenMemHandle");
    *dptr = p;
    return RTCG_OK;
}

int rtcg_ipc_close_handle(uint64_t dptr) {
    NEED_CONTEXT();
    CU_CALL(g_drv.cuIpcCloseMemHandle(dptr), "cuIpcCloseMemHandle");
    return RTCG_OK;
}

int rtcg_device_can_access_peer(int device, int peer, int *can) {
    int st = driver_ready();
    if (st != RTCG_OK) return st;
    if (!can) return fail(RTCG_ERR_INVALID, "rtcg_device_can_access_peer: null result");
    CUdevice a, b;
    CU_CALL(g_drv.cuDeviceGet(&a, device), "cuDeviceGet");
    CU_CALL(g_drv.cuDeviceGet(&b, peer), "cuDeviceGet");
    if (device == peer) { *can = 1; return RTCG_OK; }
    CU_CALL(g_drv.cuDeviceCanAccessPeer(can, a, b), "cuDeviceCanAccessPeer");
    return RTCG_OK;
}
