"""Does dynamic chunk scheduling shorten a single (isolated) dot launch?

The product reduction gives CTA b the fixed slice [b*n/G, (b+1)*n/G)
(rtcg::partition<contiguous>): an isolated 2^28 f32 dot launch takes ~302 us
against ~286 us per step when launches overlap.  Part of the gap is the
tail -- CTAs on slower memory paths finish late while finished SMs idle.
Stand-ins over the same bytes (2^28 float x, y; float4 loads, 4 in flight
per array per thread; f32 products accumulated in f64; no final fold):

  stat   : the static contiguous partition, grid = waves x resident CTAs,
           with per-CTA start / end stamps (the tail spread);
  dyncta : persistent CTAs take CH-element chunks from an atomic counter
           (next chunk fetched one ahead), one f64 partial per chunk
           (deterministic: partial[c] depends only on c);
  dynwarp: the same per warp (no __syncthreads per chunk).

Isolated = one launch bracketed by events with a synchronisation between
launches (median of 25); burst = 20 back-to-back launches / 20."""
import ctypes
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, jit  # noqa: E402

SRC = r'''
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int U>
__device__ __forceinline__ double steps(const float4 *__restrict__ x, const float4 *__restrict__ y,
                                        long c, long stride, long hi, double acc) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long k = c + u * stride;
        if (k < hi) { a[u] = __ldg(x + k); b[u] = __ldg(y + k); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long k = c + u * stride;
        if (k < hi) {
            acc += (double)__fmul_rn(a[u].x, b[u].x); acc += (double)__fmul_rn(a[u].y, b[u].y);
            acc += (double)__fmul_rn(a[u].z, b[u].z); acc += (double)__fmul_rn(a[u].w, b[u].w);
        }
    }
    return acc;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double block_sum(double v, double *red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;
}

extern "C" __global__ void __launch_bounds__(256)
stat_dot(const float4 *__restrict__ x, const float4 *__restrict__ y, long n4,
         double *partials, unsigned long long *stamps)
{
    __shared__ double red[32];
    const unsigned long long t0 = gt();
    const unsigned long g = gridDim.x, b = blockIdx.x;
    const long lo = (long)(b * (unsigned long)n4 / g), hi = (long)((b + 1) * (unsigned long)n4 / g);
    double acc = 0.0;
    for (long c = lo + threadIdx.x; c < hi; c += 4 * (long)blockDim.x)
        acc = steps<4>(x, y, c, blockDim.x, hi, acc);
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) {
        partials[b] = acc;
        stamps[2 * b] = t0;
        stamps[2 * b + 1] = gt();
    }
}

extern "C" __global__ void __launch_bounds__(256)
dyncta_dot(const float4 *__restrict__ x, const float4 *__restrict__ y, long n4, long ch4,
           unsigned nch, double *partials, unsigned *ctr)
{
    __shared__ double red[32];
    __shared__ unsigned next[2];
    if (threadIdx.x == 0) next[0] = atomicAdd(ctr, 1u);
    __syncthreads();
    int p = 0;
    unsigned ch = next[0];
    while (ch < nch) {
        if (threadIdx.x == 0) next[p ^ 1] = atomicAdd(ctr, 1u);
        const long lo = (long)ch * ch4, hi = min(lo + ch4, n4);
        double acc = 0.0;
        for (long c = lo + threadIdx.x; c < hi; c += 4 * (long)blockDim.x)
            acc = steps<4>(x, y, c, blockDim.x, hi, acc);
        acc = block_sum(acc, red);           // its __syncthreads also publish next[p ^ 1]
        if (threadIdx.x == 0) partials[ch] = acc;
        p ^= 1;
        ch = next[p];
    }
}

extern "C" __global__ void __launch_bounds__(256)
dynpdl_dot(const float4 *__restrict__ x, const float4 *__restrict__ y, long n4, long ch4,
           unsigned nch, double *partials, unsigned *ctrs, int launch)
{
    asm volatile("griddepcontrol.launch_dependents;");
    unsigned *ctr = ctrs + launch;
    double *part = partials + (long)(launch & 1) * nch;
    __shared__ double red[32];
    __shared__ unsigned next[2];
    if (threadIdx.x == 0) next[0] = atomicAdd(ctr, 1u);
    __syncthreads();
    int p = 0;
    unsigned ch = next[0];
    while (ch < nch) {
        if (threadIdx.x == 0) next[p ^ 1] = atomicAdd(ctr, 1u);
        const long lo = (long)ch * ch4, hi = min(lo + ch4, n4);
        double acc = 0.0;
        for (long c = lo + threadIdx.x; c < hi; c += 4 * (long)blockDim.x)
            acc = steps<4>(x, y, c, blockDim.x, hi, acc);
        acc = block_sum(acc, red);
        if (threadIdx.x == 0) part[ch] = acc;
        p ^= 1;
        ch = next[p];
    }
}

extern "C" __global__ void __launch_bounds__(256)
dynwarp_dot(const float4 *__restrict__ x, const float4 *__restrict__ y, long n4, long ch4,
            unsigned nch, double *partials, unsigned *ctr)
{
    const int lane = threadIdx.x & 31;
    unsigned ch = 0;
    if (lane == 0) ch = atomicAdd(ctr, 1u);
    ch = __shfl_sync(0xffffffffu, ch, 0);
    while (ch < nch) {
        unsigned nx = 0;
        if (lane == 0) nx = atomicAdd(ctr, 1u);
        const long lo = (long)ch * ch4, hi = min(lo + ch4, n4);
        double acc = 0.0;
        for (long c = lo + lane; c < hi; c += 4 * 32)
            acc = steps<4>(x, y, c, 32, hi, acc);
        acc = warp_sum(acc);
        if (lane == 0) partials[ch] = acc;
        ch = __shfl_sync(0xffffffffu, nx, 0);
    }
}
'''


def main():
    rt.set_device(0)
    mod = jit.compile(SRC)
    fns = {k: jit.get_kernel(mod, f"{k}_dot").function(0)
           for k in ("stat", "dyncta", "dynwarp", "dynpdl")}
    n = 1 << 28
    n4 = n // 4
    x, y = rt.mem_alloc(n * 4), rt.mem_alloc(n * 4)
    rt.memset_async(x, 0x3c, n * 4)
    rt.memset_async(y, 0x3d, n * 4)
    sms = rt.device_info(0)["sm_count"]
    partials = rt.mem_alloc(8 << 20)
    stamps = rt.mem_alloc(16 << 16)
    ctrs = rt.mem_alloc(4 * 64)
    rt.synchronize()
    nbytes = 8 * n
    out = {}

    def run(name, fn, grid, vals, iso_reps=25, burst=20, reset=False, block=256):
        params = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
        iso = []
        for _ in range(3):                       # warm-up
            if reset:
                rt.memset_async(ctrs, 0, 4)
            rt.launch(fn, grid, block, params)
        rt.synchronize()
        for _ in range(iso_reps):
            if reset:
                rt.memset_async(ctrs, 0, 4)
            rt.synchronize()
            s, e = rt.Event(), rt.Event()
            s.record()
            rt.launch(fn, grid, block, params)
            e.record()
            e.synchronize()
            iso.append(s.elapsed_ms(e))
        # burst: counters reset by a memset before each launch (stat needs none)
        s, e = rt.Event(), rt.Event()
        s.record()
        for _ in range(burst):
            if reset:
                rt.memset_async(ctrs, 0, 4)
            rt.launch(fn, grid, block, params)
        e.record()
        e.synchronize()
        b = s.elapsed_ms(e) / burst
        med = statistics.median(iso)
        out[name] = {"grid": grid, "isolated_us": round(med * 1e3, 1),
                     "isolated_min_us": round(min(iso) * 1e3, 1),
                     "isolated_gbs": round(nbytes / (med * 1e-3) / 1e9, 1),
                     "burst_us": round(b * 1e3, 1), "burst_gbs": round(nbytes / (b * 1e-3) / 1e9, 1)}

    occ = rt.occupancy(fns["stat"], 256, 0)
    for waves in (() if "--product-only" in sys.argv else (1, 2, 4)):
        grid = sms * occ * waves
        vals = [ctypes.c_uint64(x), ctypes.c_uint64(y), ctypes.c_int64(n4),
                ctypes.c_uint64(partials), ctypes.c_uint64(stamps)]
        run(f"stat_waves{waves}", fns["stat"], grid, vals)
        host = (ctypes.c_uint64 * (2 * grid))()
        rt.memcpy_dtoh(ctypes.addressof(host), stamps, ctypes.sizeof(host))
        rt.synchronize()
        t0 = min(host[0::2])
        ends = sorted((v - t0) / 1e3 for v in host[1::2])
        out[f"stat_waves{waves}"].update(
            first_end_us=round(ends[0], 1), median_end_us=round(ends[len(ends) // 2], 1),
            p90_end_us=round(ends[int(0.9 * len(ends))], 1), last_end_us=round(ends[-1], 1))
        print(f"stat_waves{waves}", json.dumps(out[f"stat_waves{waves}"]), flush=True)
    for kind in (() if "--product-only" in sys.argv else ("dyncta", "dynwarp")):
        occ_k = rt.occupancy(fns[kind], 256, 0)
        chunks = (1 << 12, 1 << 13, 1 << 14, 1 << 15, 1 << 16, 1 << 18) if kind == "dyncta" \
            else (1 << 12, 1 << 13, 1 << 14)
        for ch in chunks:
            ch4 = ch // 4
            nch = (n4 + ch4 - 1) // ch4
            vals = [ctypes.c_uint64(x), ctypes.c_uint64(y), ctypes.c_int64(n4),
                    ctypes.c_int64(ch4), ctypes.c_uint32(nch), ctypes.c_uint64(partials),
                    ctypes.c_uint64(ctrs)]
            name = f"{kind}_chunk{ch}"
            run(name, fns[kind], sms * occ_k, vals, reset=True)
            print(name, json.dumps(out[name]), flush=True)
            if kind == "dyncta":
                name += "_block128"
                run(name, fns[kind], sms * rt.occupancy(fns[kind], 128, 0), vals, reset=True,
                    block=128)
                print(name, json.dumps(out[name]), flush=True)
    # dynamic chunks with programmatic dependent launch (per-launch counters,
    # zeroed before the burst): the overlapped rate to compare with the
    # product's burst_pdl_us
    occ_p = rt.occupancy(fns["dynpdl"], 256, 0)
    for ch in (() if "--product-only" in sys.argv else (1 << 13, 1 << 14)):
        ch4 = ch // 4
        nch = (n4 + ch4 - 1) // ch4
        best = float("inf")
        for _ in range(3):
            rt.memset_async(ctrs, 0, 4 * 64)
            rt.synchronize()
            s_, e_ = rt.Event(), rt.Event()
            s_.record()
            for k in range(20):
                vals = [ctypes.c_uint64(x), ctypes.c_uint64(y), ctypes.c_int64(n4),
                        ctypes.c_int64(ch4), ctypes.c_uint32(nch), ctypes.c_uint64(partials),
                        ctypes.c_uint64(ctrs), ctypes.c_int32(k)]
                params = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
                rt.launch_overlapped(fns["dynpdl"], sms * occ_p, 256, params)
            e_.record()
            e_.synchronize()
            best = min(best, s_.elapsed_ms(e_) / 20)
        name = f"dynpdl_chunk{ch}"
        out[name] = {"grid": sms * occ_p, "burst_pdl_us": round(best * 1e3, 1),
                     "burst_pdl_gbs": round(nbytes / (best * 1e-3) / 1e9, 1)}
        print(name, json.dumps(out[name]), flush=True)

    # the product kernel on the same bytes (public API, isolated and overlapped)
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    pool = nd.MemoryPool(device=0)
    gx, gy = pool.alloc(nd.float32, (n,)), pool.alloc(nd.float32, (n,))
    rt.memset_async(gx.gpudata, 0x3c, n * 4)
    rt.memset_async(gy.gpudata, 0x3d, n * 4)
    o = pool.alloc(nd.float32, ())
    for block, unroll, waves, chunk in ((128, 4, 2, 0), (256, 4, 2, 0), (512, 1, 2, 0),
                                        (1024, 1, 2, 0), (256, 4, 1, 8192), (256, 4, 1, 4096),
                                        (256, 4, 1, 16384), (128, 4, 1, 8192),
                                        (512, 1, 1, 8192), (256, 4, 2, 8192)):
        k = rd.ReductionKernel(rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b",
                                                "x[i] * y[i]"), "dot_k",
                               ew.VariantParams(block=block, unroll=unroll, waves=waves,
                                                chunk=chunk))
        for _ in range(3):
            k.launch(gx, gy, out=o)
        rt.synchronize()
        iso = []
        for _ in range(25):
            rt.synchronize()
            s, e = rt.Event(), rt.Event()
            s.record()
            k.launch(gx, gy, out=o)
            e.record()
            e.synchronize()
            iso.append(s.elapsed_ms(e))
        res = {}
        for ov in (False, True):
            s, e = rt.Event(), rt.Event()
            s.record()
            for _ in range(20):
                k.launch(gx, gy, out=o, overlap_previous=ov)
            e.record()
            e.synchronize()
            res["pdl" if ov else "serial"] = s.elapsed_ms(e) / 20
        med = statistics.median(iso)
        name = f"product_b{block}_u{unroll}_w{waves}" + (f"_chunk{chunk}" if chunk else "")
        out[name] = {"isolated_us": round(med * 1e3, 1), "isolated_min_us": round(min(iso) * 1e3, 1),
                     "isolated_gbs": round(nbytes / (med * 1e-3) / 1e9, 1),
                     "burst_serial_us": round(res["serial"] * 1e3, 1),
                     "burst_pdl_us": round(res["pdl"] * 1e3, 1)}
        print(name, json.dumps(out[name]), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/probe_dynamic_chunks.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
