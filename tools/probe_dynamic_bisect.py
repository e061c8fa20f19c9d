"""Where does the product's dynamic-chunk dot lose to the stand-in?

The generated dynamic entry (VariantParams(block=256, unroll=4, chunk=8192))
compiled as is and with parts cut out, launched by hand on 2^28 f32 x, y
(serial seq, counter at ticket[7], the ticket block zeroed before every
launch for every variant):

  P   the generated kernel
  A   without rtcg::chunk_counter (no slot wait / griddepcontrol.wait)
  B   without the final rtcg::finish (no arrival, no last-CTA fold)
  AB  both cut
  C   finish folding one partial instead of every chunk's (timing only)
(D, a contiguous run per thread with 16 __ldcg loads in flight, measured
level with P when P still folded contiguous runs: the loads were
uncoalesced, one sector per lane; P now folds strided, coalesced runs.)

isolated_us = median of 15 event-bracketed launches, serial_us = 20
launches (each after a memset) / 20."""
import ctypes
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, jit  # noqa: E402
from paper_0911_3456_b200 import ndarray as nd, reduction as rd  # noqa: E402


def main():
    rt.set_device(0)
    spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
    src = rd.generate_reduction_source(spec, "dot_k", ew.VariantParams(block=256, unroll=4,
                                                                      chunk=8192),
                                       entries="vector")
    counter = "unsigned *const rtcg_ctr = rtcg::chunk_counter(rtcg_ticket, rtcg_seq);"
    assert counter in src
    fin_at = src.index("    rtcg::finish(RTCG_NEUTRAL, RTCG_NEUTRAL")
    fin_end = src.index("plan.count);", fin_at) + len("plan.count);")
    cut_a = src.replace(counter, "unsigned *const rtcg_ctr = rtcg_ticket + 7;")
    variants = {"P": src, "A": cut_a,
                "B": src[:fin_at] + src[fin_end:],
                "AB": cut_a[:cut_a.index("    rtcg::finish(RTCG_NEUTRAL, RTCG_NEUTRAL")] +
                cut_a[cut_a.index("plan.count);", cut_a.index("    rtcg::finish(RTCG_NEUTRAL"))
                      + len("plan.count);"):]}
    variants["C"] = src.replace("rtcg_seq,\n                 plan.count);", "rtcg_seq,\n                 1u);")
    assert variants["C"] != src
    fns = {}
    for k, s in variants.items():
        fns[k] = jit.get_kernel(jit.compile(s), "dot_k").function(0)
    n = 1 << 28
    x, y = rt.mem_alloc(n * 4), rt.mem_alloc(n * 4)
    rt.memset_async(x, 0x3c, n * 4)
    rt.memset_async(y, 0x3d, n * 4)
    partials = rt.mem_alloc(3 * 65536 * 8)
    block = rt.mem_alloc(64)
    sms = rt.device_info(0)["sm_count"]
    rt.synchronize()
    out = {}
    for rep in range(2):
        for k, fn in fns.items():
            grid = sms * rt.occupancy(fn, 256, 0)
            vals = [ctypes.c_uint64(x), ctypes.c_uint64(y), ctypes.c_long(0), ctypes.c_long(n),
                    ctypes.c_uint64(partials + 2 * 65536 * 8), ctypes.c_uint64(block),
                    ctypes.c_uint64(block + 16), ctypes.c_uint64(block + 32),
                    ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint64(1 << 63)]
            params = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
            iso = []
            for _ in range(15):
                rt.memset_async(block + 32, 0, 32)
                rt.synchronize()
                s, e = rt.Event(), rt.Event()
                s.record()
                rt.launch(fn, grid, 256, params)
                e.record()
                e.synchronize()
                iso.append(s.elapsed_ms(e) * 1e3)
            s, e = rt.Event(), rt.Event()
            s.record()
            for _ in range(20):
                rt.memset_async(block + 32, 0, 32)
                rt.launch(fn, grid, 256, params)
            e.record()
            e.synchronize()
            out.setdefault(k, []).append({"grid": grid, "isolated_us": round(statistics.median(iso), 1),
                                          "serial_us": round(s.elapsed_ms(e) * 1e3 / 20, 1)})
    print(json.dumps({"what": __doc__.split("\n\n")[0], "rows": out}, indent=1))


if __name__ == "__main__":
    main()
