"""Does programmatic dependent launch hide a long tail in the last CTA?

A stand-in for the reduction kernel: every CTA triggers its dependents at
start, streams a share of 2^25 float4s, waits on the previous grid
(griddepcontrol.wait, as rtcg::finish does), takes a ticket; the last CTA
then spins for EXTRA ns (the stand-in for the fold + cross-GPU exchange).
Six back-to-back overlapped launches, CUDA-event time, for EXTRA = 0 / 5 /
20 us and grids of 1 and 2 resident waves.  Per-CTA globaltimer stamps show
when launch k+1's CTAs start relative to launch k's end."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, jit  # noqa: E402

SRC = r'''
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
extern "C" __global__ void __launch_bounds__(256)
pdl_probe(const float4 *__restrict__ x, long n4, unsigned long long *stamps, int launch,
          unsigned *tickets, long long extra_ns, float *sink, int wait_last)
{
    asm volatile("griddepcontrol.launch_dependents;");
    const unsigned long long t0 = gt();
    float acc = 0.f;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (long)gridDim.x * blockDim.x) {
        const float4 v = __ldg(x + i);
        acc += v.x + v.y + v.z + v.w;
    }
    const unsigned long long t1 = gt();
    if (!wait_last) asm volatile("griddepcontrol.wait;" ::: "memory");
    const unsigned long long t2 = gt();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(tickets + launch, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && wait_last) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (last && threadIdx.x == 0) {
        const unsigned long long s = gt();
        while ((long long)(gt() - s) < extra_ns) { }
    }
    const unsigned long long t3 = gt();
    if (threadIdx.x == 0) {
        unsigned long long *p = stamps + ((long)launch * gridDim.x + blockIdx.x) * 4;
        p[0] = t0; p[1] = t1; p[2] = t2; p[3] = t3;
    }
    if (acc == 1.2345e-30f) *sink = acc;
}
'''


def main():
    rt.set_device(0)
    mod = jit.compile(SRC)
    fn = jit.get_kernel(mod, "pdl_probe").function(0)
    n4 = (1 << 25) // 4 * 2            # 2^25 floats x2 (a dot share's bytes)
    x = rt.mem_alloc(n4 * 16)
    rt.memset_async(x, 0, n4 * 16)
    sms = rt.device_info(0)["sm_count"]
    occ = rt.occupancy(fn, 256, 0)
    launches = 6
    out = {}
    for waves, wait_last in ((1, 0), (2, 0), (1, 1), (2, 1)):
        grid = sms * occ * waves
        stamps = rt.mem_alloc(launches * grid * 4 * 8)
        tickets = rt.mem_alloc(4 * launches)
        sink = rt.mem_alloc(4)
        for extra_us in (0, 5, 20):
            for overlap in ((True,) if wait_last else (False, True)):
                best, tl = float("inf"), None
                for _ in range(3):
                    rt.memset_async(tickets, 0, 4 * launches)
                    rt.synchronize()
                    vals = [ctypes.c_uint64(x), ctypes.c_int64(n4), ctypes.c_uint64(stamps),
                            ctypes.c_int32(0), ctypes.c_uint64(tickets),
                            ctypes.c_int64(extra_us * 1000), ctypes.c_uint64(sink),
                            ctypes.c_int32(wait_last)]
                    s, e = rt.Event(), rt.Event()
                    s.record()
                    for k in range(launches):
                        vals[3] = ctypes.c_int32(k)
                        params = (ctypes.c_void_p * len(vals))(
                            *[ctypes.addressof(v) for v in vals])
                        (rt.launch_overlapped if overlap else rt.launch)(fn, grid, 256, params)
                    e.record()
                    e.synchronize()
                    ms = s.elapsed_ms(e)
                    if ms < best:
                        best = ms
                        host = (ctypes.c_uint64 * (launches * grid * 4))()
                        rt.memcpy_dtoh(ctypes.addressof(host), stamps, ctypes.sizeof(host))
                        rt.synchronize()
                        tl = []
                        for k in range(launches):
                            rows = [host[(k * grid + b) * 4:(k * grid + b) * 4 + 4]
                                    for b in range(grid)]
                            tl.append((min(r[0] for r in rows), max(r[3] for r in rows)))
                base = tl[0][0]
                key = (f"waves{waves}_{'waitlast' if wait_last else 'waitall'}_extra{extra_us}us_"
                       f"{'pdl' if overlap else 'serial'}")
                out[key] = {"us_per_launch": round(best * 1e3 / launches, 2),
                            "launch_start_end_us": [(round((a - base) / 1e3, 1),
                                                     round((b - base) / 1e3, 1)) for a, b in tl]}
                print(key, json.dumps(out[key]), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/probe_pdl_tail.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
