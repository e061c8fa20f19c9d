"""Small-n reductions: one thread-block cluster with a distributed-shared-
memory fold vs the package's multi-CTA single-pass reduction (partials +
arrival ticket + last-CTA fold).

The cluster kernel: G CTAs (one cluster, __cluster_dims__) of 1024 threads
stream the input with U 16-byte loads in flight per thread, fold each CTA in
shared memory, then CTA 0 reads the G per-CTA partials through DSMEM
(mapa + ld.shared::cluster) after a cluster barrier and folds them in CTA
order -- no global partials, no atomics, no gpu-scope fences.  float32 sum
with a double accumulator, like the package's sum kernel.  Device time per
kernel from CUDA graphs of 50 back-to-back launches; results are printed.

    python tools/probe_cluster_reduction.py [--out gpurun_out/probe_cluster_reduction.json]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, reduction as rd, graph  # noqa: E402

SRC = r'''
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned smem_addr(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
template <int G, int U>
__device__ __forceinline__ void cluster_sum(const float4 *__restrict__ x, long nv, double *out) {
    __shared__ double warp_part[32];
    __shared__ double cta_part;
    const unsigned rank = blockIdx.x % G;          // one cluster: rank == blockIdx.x
    const long t = (long)rank * blockDim.x + threadIdx.x;
    const long step = (long)G * blockDim.x;
    double acc = 0.0;
    for (long c = t; c < nv; c += U * step) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c + u * step < nv) v[u] = __ldg(x + c + u * step);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c + u * step < nv)
                acc = acc + (double)v[u].x + (double)v[u].y + (double)v[u].z + (double)v[u].w;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = threadIdx.x < (blockDim.x >> 5) ? warp_part[threadIdx.x] : 0.0;
        w = warp_sum(w);
        if (threadIdx.x == 0) cta_part = w;
    }
    // publish cta_part to the cluster; CTA 0 folds the G partials in order
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
        double r = 0.0;
        const unsigned local = smem_addr(&cta_part);
#pragma unroll
        for (unsigned g = 0; g < G; ++g) {
            unsigned remote;
            double v;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(g));
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
            r += v;
        }
        out[0] = r;
    }
    // keep every CTA's shared memory alive until CTA 0 has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
extern "C" __global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024)
csum8_u1(const float4 *x, long nv, double *out) { cluster_sum<8, 1>(x, nv, out); }
extern "C" __global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024)
csum8_u4(const float4 *x, long nv, double *out) { cluster_sum<8, 4>(x, nv, out); }
extern "C" __global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(1024)
csum4_u4(const float4 *x, long nv, double *out) { cluster_sum<4, 4>(x, nv, out); }
extern "C" __global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024)
csum8_u8(const float4 *x, long nv, double *out) { cluster_sum<8, 8>(x, nv, out); }
'''


def graph_us(launch, per_graph=50, replays=20):
    """Device time per kernel: ``per_graph`` launches captured in one graph,
    replayed ``replays`` times (no host launch cost in the measurement)."""
    g = graph.Graph()
    with rt.use_stream(g.stream):
        launch()
        g.synchronize()
    with g.capture():
        for _ in range(per_graph):
            launch()
    g.launch()
    g.synchronize()
    s, e = rt.Event(), rt.Event()
    s.record(g.stream.handle)
    for _ in range(replays):
        g.launch()
    e.record(g.stream.handle)
    e.synchronize()
    return s.elapsed_ms(e) / (replays * per_graph) * 1e3


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default="gpurun_out/probe_cluster_reduction.json")
    a = p.parse_args()
    rt.set_device(0)
    img, _ = rt.compile_cubin(SRC, ["-arch=sm_100a", "-fmad=false", "-std=c++17"])
    mod = rt.Module(img)
    pool = nd.MemoryPool(device=0)
    rows = []
    sk = rd.sum_kernel(nd.float32)
    for lg in (12, 14, 16, 17, 18, 20):
        n = 1 << lg
        hx = np.random.default_rng(lg).uniform(-1, 1, n).astype(np.float32)
        x = nd.from_host(pool, nd.float32, hx)
        o = pool.alloc(nd.float32, ())
        want = float(np.float32(np.sum(hx.astype(np.float64))))
        row = {"n": f"2^{lg}", "package_sum_us": round(graph_us(lambda: sk.launch(x, out=o)), 2),
               "package_sum": float(o.get()), "want": want}
        out = pool.alloc(nd.float64, (1,))
        for name, g in (("csum4_u4", 4), ("csum8_u1", 8), ("csum8_u4", 8), ("csum8_u8", 8)):
            fn = mod.function(name)
            vals = [ctypes.c_uint64(x.address), ctypes.c_long(n // 4), ctypes.c_uint64(out.address)]
            params = (ctypes.c_void_p * 3)(*[ctypes.addressof(v) for v in vals])
            row[f"{name}_us"] = round(graph_us(lambda: rt.launch(fn, g, 1024, params)), 2)
            row[f"{name}_result"] = float(np.float32(out.get()[0]))
        rows.append(row)
        print(json.dumps(row), flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
