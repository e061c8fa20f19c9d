"""A/B of the reduction's arrival protocol in ``rtcg::finish``.

  old: partials[b] = acc; __threadfence(); atomicAdd(ticket)   (MEMBAR.SC.GPU)
       ... last CTA: __threadfence() again before reading the partials
  new: partials[b] = acc; atom.add.acq_rel.gpu(ticket)          (MEMBAR.ALL.GPU)
       ... last CTA reads after the barrier, no second fence

Both builds in one process (the old one from the prelude text with the new
block swapped back), float32 sum / max / dot; per size: a CUDA graph of 20
serial launches replayed (device time per launch, no host path), and 20
back-to-back overlapped launches (the bench's protocol).  Five alternating
rounds, best of each.

    python tools/probe_finish_fences.py [fences|division] > gpurun_out/finish_fences.json

(``division``: the last CTA's partial ranges with 32-bit instead of 64-bit
division, the same values.)
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_0911_3456_b200 import _codegen as cg, _runtime as rt, graph  # noqa: E402
from paper_0911_3456_b200 import ndarray as nd, reduction as rd  # noqa: E402

DIV_NEW = """    // thread t folds partials [t*g/b, (t+1)*g/b); 32-bit division whenever
    // (t+1)*g fits (g < 2^22 -- every practical grid), 64-bit otherwise
    const unsigned g = gridDim.x, b = blockDim.x, t = threadIdx.x;
    unsigned long lo, hi;
    if (g < (1u << 22)) {
        lo = t * g / b;
        hi = (t + 1) * g / b;
    } else {
        lo = (unsigned long)t * g / b;
        hi = (unsigned long)(t + 1) * g / b;
    }
"""
DIV_OLD = """    const unsigned long g = gridDim.x, b = blockDim.x, t = threadIdx.x;
    const unsigned long lo = t * g / b, hi = (t + 1) * g / b;
"""
NEW = """        last_cta = atom_add_acq_rel_gpu_u32(ticket + slot, 1u) == gridDim.x - 1;
    }
    __syncthreads();        // thread 0's acquire orders the whole CTA's loads
    if (!last_cta) return;
    if (!serial) asm volatile("griddepcontrol.wait;" ::: "memory");
"""
OLD = """        __threadfence();
        last_cta = atomicAdd(ticket + slot, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last_cta) return;
    if (!serial) asm volatile("griddepcontrol.wait;" ::: "memory");
    __threadfence();
"""


WHAT = sys.argv[1] if len(sys.argv) > 1 else "fences"


def build(old: bool):
    real = cg.template

    def patched(name):
        text = real(name)
        if name == "prelude.cuh" and old:
            a, b = (DIV_NEW, DIV_OLD) if WHAT == "division" else (NEW, OLD)
            assert a in text
            text = text.replace(a, b)
        return text
    cg.template = patched
    try:
        tag = ("old" if old else "new") + WHAT[:3]
        return {"sum": rd.ReductionKernel(rd.ReductionSpec("float *x", nd.float32, "0", "a + b",
                                                           None), f"sum_{tag}"),
                "max": rd.ReductionKernel(rd.ReductionSpec("float *x", nd.float32, "-INFINITY",
                                                           "a > b ? a : b", None), f"max_{tag}"),
                "dot": rd.ReductionKernel(rd.ReductionSpec("float *x, float *y", nd.float32, "0",
                                                           "a + b", "x[i] * y[i]"), f"dot_{tag}")}
    finally:
        cg.template = real


def graph_us(fn, reps=20, replays=20):
    st = rt.Stream()
    with rt.use_stream(st.handle):
        fn()
        st.synchronize()
        g = graph.Graph(st)
        with g.capture():
            for _ in range(reps):
                fn()
        g.launch()
        st.synchronize()
        s, e = rt.Event(), rt.Event()
        s.record(st.handle)
        for _ in range(replays):
            g.launch()
        e.record(st.handle)
        e.synchronize()
    g.close()
    return s.elapsed_ms(e) * 1e3 / (reps * replays)


def burst_us(fn, reps=20):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_ms(e) * 1e3 / reps


def main():
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    kernels = {"old": build(True), "new": build(False)}
    rng = np.random.default_rng(0)
    res = {}
    for lg in (12, 16, 20, 24, 28):
        n = 1 << lg
        x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
        y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
        o = pool.alloc(nd.float32, ())
        row = {}
        for name in ("sum", "max", "dot"):
            args = (x, y) if name == "dot" else (x,)
            vals = {k: float(kernels[k][name](*args)) for k in kernels}
            assert vals["old"] == vals["new"], (name, lg, vals)
            best = {}
            for _ in range(5):
                for tag in ("old", "new"):
                    k = kernels[tag][name]
                    g = graph_us(lambda k=k: k.launch(*args, out=o))
                    b = burst_us(lambda k=k: k.launch(*args, out=o, overlap_previous=True))
                    cur = best.setdefault(tag, {"graph_serial_us": g, "burst_overlapped_us": b})
                    cur["graph_serial_us"] = min(cur["graph_serial_us"], g)
                    cur["burst_overlapped_us"] = min(cur["burst_overlapped_us"], b)
            row[name] = {t: {k: round(v, 3) for k, v in d.items()} for t, d in best.items()}
            row[name]["same_result"] = True
        res[f"2^{lg}"] = row
        for a in (x, y, o):
            a.free()
    print(json.dumps({"what": __doc__.split("\n\n")[0], "rows": res}, indent=1))


if __name__ == "__main__":
    main()
