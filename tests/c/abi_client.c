/* A C client of librtcg_b200.so through include/rtcg_b200.h only -- what a
 * non-Python host (the reference's ctypes seam, a cgo/JNI binding) would do:
 * NVRTC-compile a generated-style kernel with the reference ABI shape
 * (pointers + widened scalars + long start/end), load it, launch it over
 * [0, n), copy back and check against a host loop.
 *
 *   abi_client compile   -- NVRTC only (works without a GPU)
 *   abi_client run       -- compile + load + launch + verify on device 0
 * Exit status 0 = pass; messages on stderr. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rtcg_b200.h"

static const char *SOURCE =
    "extern \"C\" __global__ void axpy_c(double wa, const float *x, double wb,\n"
    "                                    const float *y, float *z, long start, long end)\n"
    "{\n"
    "    const float a = (float) wa, b = (float) wb;\n"
    "    for (long i = start + (long) blockIdx.x * blockDim.x + threadIdx.x; i < end;\n"
    "         i += (long) gridDim.x * blockDim.x)\n"
    "        z[i] = a * x[i] + b * y[i];\n"
    "}\n";

#define CHECK(call)                                                              \
    do {                                                                         \
        int st_ = (call);                                                        \
        if (st_ != RTCG_OK) {                                                    \
            fprintf(stderr, "%s -> %d: %s\n", #call, st_, rtcg_last_error());    \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main(int argc, char **argv) {
    const int run = argc > 1 && strcmp(argv[1], "run") == 0;
    if (rtcg_abi_version() != RTCG_ABI_VERSION) return 2;
    int major = 0, minor = 0;
    CHECK(rtcg_nvrtc_version(&major, &minor));
    const char *opts[] = {"-arch=sm_100a", "-fmad=false"};
    void *image = NULL;
    size_t size = 0;
    char *log = NULL;
    CHECK(rtcg_compile(SOURCE, "abi_client.cu", opts, 2, &image, &size, &log));
    rtcg_free_buffer(log);
    if (size < 4 || memcmp(image, "\x7f" "ELF", 4) != 0) return 3;
    /* a compile error must come back as a status + log, not a crash */
    void *bad = NULL;
    size_t bad_size = 0;
    char *bad_log = NULL;
    if (rtcg_compile("not cuda", "bad.cu", opts, 2, &bad, &bad_size, &bad_log) !=
        RTCG_ERR_COMPILE || !bad_log || !strstr(bad_log, "error"))
        return 4;
    rtcg_free_buffer(bad_log);
    printf("nvrtc %d.%d: cubin %zu bytes\n", major, minor, size);
    if (!run) {
        rtcg_free_buffer(image);
        return 0;
    }

    CHECK(rtcg_set_device(0));
    rtcg_module_t module;
    rtcg_function_t fn;
    CHECK(rtcg_module_load(image, size, &module));
    rtcg_free_buffer(image);
    CHECK(rtcg_module_function(module, "axpy_c", &fn));
    if (rtcg_module_function(module, "no_such_kernel", &fn) != RTCG_ERR_NOT_FOUND) return 5;
    CHECK(rtcg_module_function(module, "axpy_c", &fn));

    const long n = (1L << 20) + 3;
    const uint64_t bytes = (uint64_t) n * sizeof(float);
    float *hx = malloc(bytes), *hy = malloc(bytes), *hz = malloc(bytes);
    for (long i = 0; i < n; ++i) {
        hx[i] = (float) ((i * 7919) % 2001 - 1000) / 1000.0f;
        hy[i] = (float) ((i * 104729) % 2001 - 1000) / 999.0f;
    }
    uint64_t dx, dy, dz;
    CHECK(rtcg_mem_alloc(bytes, &dx));
    CHECK(rtcg_mem_alloc(bytes, &dy));
    CHECK(rtcg_mem_alloc(bytes, &dz));
    CHECK(rtcg_copy_htod(dx, hx, bytes, NULL));
    CHECK(rtcg_copy_htod(dy, hy, bytes, NULL));
    /* kernel parameters: a pack of pointers to values, like the reference's
     * void **args (scalars widened to double, as src/elementwise.py:316-321) */
    double wa = 2.0, wb = -3.0;
    long start = 0, end = n;
    void *params[] = {&wa, &dx, &wb, &dy, &dz, &start, &end};
    /* launch on a private stream ordered after the uploads on the legacy
     * stream (what the streamed host calls do with the caller's stream) */
    rtcg_stream_t stream;
    rtcg_event_t uploaded;
    CHECK(rtcg_stream_create(&stream));
    CHECK(rtcg_event_create(&uploaded));
    CHECK(rtcg_event_record(uploaded, NULL));
    CHECK(rtcg_stream_wait_event(stream, uploaded));
    CHECK(rtcg_launch(fn, 592, 256, 0, stream, params));
    CHECK(rtcg_copy_dtoh(hz, dz, bytes, stream));
    CHECK(rtcg_stream_synchronize(stream));
    CHECK(rtcg_event_destroy(uploaded));
    CHECK(rtcg_stream_destroy(stream));
    char bus[32];
    CHECK(rtcg_device_pci_bus_id(0, bus, (int) sizeof bus));
    if (rtcg_device_pci_bus_id(0, bus, 4) != RTCG_ERR_INVALID) return 7;
    printf("device 0 at %s\n", bus);
    long bad_count = 0;
    for (long i = 0; i < n; ++i) {
        volatile float ax = 2.0f * hx[i], by = -3.0f * hy[i];   /* no contraction */
        if (hz[i] != ax + by) ++bad_count;
    }
    CHECK(rtcg_mem_free(dx));
    CHECK(rtcg_mem_free(dy));
    CHECK(rtcg_mem_free(dz));
    CHECK(rtcg_module_unload(module));
    free(hx);
    free(hy);
    free(hz);
    printf("axpy over %ld elements: %ld mismatches\n", n, bad_count);
    return bad_count == 0 ? 0 : 6;
}
