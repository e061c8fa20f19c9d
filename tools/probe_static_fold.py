"""Static-partition reductions: does a coalesced fold of the CTA partials
shorten the launch?  The generated 2^28 f32 dot (static partition, the
bench's variants) as is -- the last CTA's thread t folds partials
[t*g/b, (t+1)*g/b) with dependent volatile loads -- against the same
kernel whose last CTA folds the strided, coalesced runs t, t + b, ... with
16 .cg loads in flight (the dynamic-chunk fold).  Launched by hand (serial
seq, slot 2), interleaved, one process; the results must agree to the
fold's rounding (the order differs).

    python tools/probe_static_fold.py > gpurun_out/probe_static_fold.json
"""
import ctypes
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, jit  # noqa: E402
from paper_0911_3456_b200 import ndarray as nd, reduction as rd  # noqa: E402

STATIC = """        const volatile T *vp = partials;
        for (unsigned long j = lo; j < hi; ++j) v = f(v, (T)vp[j]);"""
COALESCED = """        unsigned long j = t;
        for (; j + 15ul * b < g; j += 16ul * b) {
            T r[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] = ld_cg(partials + j + (unsigned long)k * b);
#pragma unroll
            for (int k = 0; k < 16; ++k) v = f(v, r[k]);
        }
        for (; j < g; j += b) v = f(v, ld_cg(partials + j));"""


def main():
    rt.set_device(0)
    spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
    n = 1 << 28
    x, y = rt.mem_alloc(n * 4), rt.mem_alloc(n * 4)
    rt.memset_async(x, 0x3c, n * 4)
    rt.memset_async(y, 0x3d, n * 4)
    partials = rt.mem_alloc(3 * 65536 * 8)
    block_mem = rt.mem_alloc(64)
    sms = rt.device_info(0)["sm_count"]
    rt.synchronize()
    kernels = {}
    for blk, unroll, waves in ((128, 1, 2), (256, 4, 2), (512, 1, 2), (1024, 1, 2)):
        src = rd.generate_reduction_source(spec, "dot_k", ew.VariantParams(
            block=blk, unroll=unroll, waves=waves), entries="vector")
        assert STATIC in src
        for kind, text in (("contiguous", src), ("coalesced", src.replace(STATIC, COALESCED))):
            fn = jit.get_kernel(jit.compile(text), "dot_k").function(0)
            kernels[(blk, unroll, waves, kind)] = (fn, sms * rt.occupancy(fn, blk, 0) * waves,
                                                  rt.registers(fn))
    rows = {}
    for _ in range(3):
        for (blk, unroll, waves, kind), (fn, grid, regs) in kernels.items():
            vals = [ctypes.c_uint64(x), ctypes.c_uint64(y), ctypes.c_long(0), ctypes.c_long(n),
                    ctypes.c_uint64(partials + 2 * 65536 * 8), ctypes.c_uint64(block_mem),
                    ctypes.c_uint64(block_mem + 16), ctypes.c_uint64(block_mem + 32),
                    ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint64(1 << 63)]
            params = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
            key = f"b{blk}_u{unroll}_w{waves}_{kind}"
            row = rows.setdefault(key, {"grid": grid, "registers": regs, "iso": [], "serial": []})
            rt.memset_async(block_mem + 32, 0, 32)
            rt.launch(fn, grid, blk, params)
            rt.synchronize()
            for _ in range(7):
                s, e = rt.Event(), rt.Event()
                s.record()
                rt.launch(fn, grid, blk, params)
                e.record()
                e.synchronize()
                row["iso"].append(s.elapsed_ms(e) * 1e3)
            s, e = rt.Event(), rt.Event()
            s.record()
            for _ in range(20):
                rt.launch(fn, grid, blk, params)
            e.record()
            e.synchronize()
            row["serial"].append(s.elapsed_ms(e) * 1e3 / 20)
            box = ctypes.c_double()
            rt.memcpy_dtoh(ctypes.addressof(box), block_mem, 8)
            rt.synchronize()
            row["result"] = box.value
    out = {k: {"grid": r["grid"], "registers": r["registers"],
               "isolated_us": round(statistics.median(r["iso"]), 1),
               "serial_us": round(min(r["serial"]), 1), "result": r["result"]}
           for k, r in rows.items()}
    print(json.dumps({"what": __doc__.split("\n\n")[0], "rows": out}, indent=1))


if __name__ == "__main__":
    main()
