"""Do 256-bit global accesses (LDG/STG.E.ENL2.256, sm_100) stream faster than
128-bit ones?  Hand-written copy / axpy / dot / f64 poly+sin at 2^28, same
grid policy, v4.b32 vs v8.b32 accesses."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd  # noqa: E402

SRC = r'''
struct v8 { float a[8]; };
template <int W> __device__ __forceinline__ void ld(float *r, const float *p) {
    if (W == 8) asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]) : "l"(p));
    else asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p));
}
template <int W> __device__ __forceinline__ void st(float *p, const float *r) {
    if (W == 8) asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
        :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
    else asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};"
        :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]) : "memory");
}
template <int W> __device__ void axpy_body(float a, const float *x, float b, const float *y, float *z, long n) {
    long step = (long)gridDim.x * blockDim.x * W;
    for (long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n; i += step) {
        float rx[8], ry[8], rz[8];
        ld<W>(rx, x + i); ld<W>(ry, y + i);
        #pragma unroll
        for (int k = 0; k < W; ++k) rz[k] = a * rx[k] + b * ry[k];
        st<W>(z + i, rz);
    }
}
template <int W> __device__ void dot_body(const float *x, const float *y, double *part, long n) {
    long step = (long)gridDim.x * blockDim.x * W;
    double acc = 0;
    for (long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n; i += step) {
        float rx[8], ry[8];
        ld<W>(rx, x + i); ld<W>(ry, y + i);
        #pragma unroll
        for (int k = 0; k < W; ++k) acc += (double)(rx[k] * ry[k]);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(part, acc);
}
extern "C" __global__ void axpy4(float a, const float *x, float b, const float *y, float *z, long n) { axpy_body<4>(a, x, b, y, z, n); }
extern "C" __global__ void axpy8(float a, const float *x, float b, const float *y, float *z, long n) { axpy_body<8>(a, x, b, y, z, n); }
extern "C" __global__ void dot4(const float *x, const float *y, double *p, long n) { dot_body<4>(x, y, p, n); }
extern "C" __global__ void dot8(const float *x, const float *y, double *p, long n) { dot_body<8>(x, y, p, n); }
'''


def main():
    rt.set_device(0)
    img, _ = rt.compile_cubin(SRC, ["-arch=sm_100a", "-fmad=false"])
    mod = rt.Module(img)
    pool = nd.MemoryPool(device=0)
    n = 1 << 28
    rng = np.random.default_rng(0)
    x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    z = pool.alloc_uninitialized(nd.float32, (n,))
    part = pool.alloc(nd.float64, (1,))
    sms = rt.device_info(0)["sm_count"]
    rows = []
    for name, nbytes, vals in (
            ("axpy", 12 * n, lambda: [ctypes.c_float(2.0), ctypes.c_uint64(x.address),
                                      ctypes.c_float(-3.0), ctypes.c_uint64(y.address),
                                      ctypes.c_uint64(z.address), ctypes.c_long(n)]),
            ("dot", 8 * n, lambda: [ctypes.c_uint64(x.address), ctypes.c_uint64(y.address),
                                    ctypes.c_uint64(part.address), ctypes.c_long(n)])):
        for w in (4, 8):
            fn = mod.function(f"{name}{w}")
            for block in (128, 256, 512):
                for grid_mult in (0, 1, 2, 4):
                    grid = (n // (block * w)) if grid_mult == 0 else \
                        sms * rt.occupancy(fn, block) * grid_mult
                    v = vals()
                    params = (ctypes.c_void_p * len(v))(*[ctypes.addressof(a) for a in v])
                    launch = lambda: rt.launch(fn, grid, block, params)  # noqa: E731
                    launch()
                    rt.synchronize()
                    s, e = rt.Event(), rt.Event()
                    s.record()
                    for _ in range(20):
                        launch()
                    e.record()
                    e.synchronize()
                    ms = s.elapsed_ms(e) / 20
                    rows.append({"kernel": name, "bits": 32 * w, "block": block,
                                 "grid": grid, "GB/s": round(nbytes / ms / 1e6)})
    for name in ("axpy", "dot"):
        for bits in (128, 256):
            best = max((r for r in rows if r["kernel"] == name and r["bits"] == bits),
                       key=lambda r: r["GB/s"])
            print(json.dumps(best), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/probe_ldg256.json").write_text(json.dumps(rows, indent=1))


main()
