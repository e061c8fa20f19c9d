"""Cost of the in-kernel peer exchange at world size 1: back-to-back dot f32
2^28 launches, local vs with a one-rank mailbox, with and without overlapped
(programmatic dependent) launches; CUDA-event time per launch (50-launch
bursts, best of 3), plus the host time per launch call."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import parallel as par, reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
out = {}
for lg in (20, 24, 28):
    n = 1 << lg
    rng = np.random.default_rng(0)
    x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    o = pool.alloc_uninitialized(nd.float32, ())
    k = rd.ReductionKernel(rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b",
                                            "x[i] * y[i]"), "dot_k",
                           ew.VariantParams(block=256, unroll=1, waves=2))
    box = par.PeerMailbox.local_group(1)[0]
    import types
    kb = rd.ReductionKernel(k.spec, "dot_k", k.variant)     # forced onto the Python binder
    kb._plan = lambda dev: types.SimpleNamespace(launch=lambda *a: None)
    print(json.dumps({"native": k.launch_config(x, y), "grid_python": kb.launch_config(x, y)}))
    cases = {"local": lambda ov: k.launch(x, y, out=o, overlap_previous=ov),
             "binder": lambda ov: kb.launch(x, y, out=o, overlap_previous=ov),
             "p2p": lambda ov: k.launch(x, y, out=o, peers=box, overlap_previous=ov)}
    row = {}
    for name, fn in cases.items():
        for ov in (False, True):
            fn(ov)
            rt.synchronize()
            best = float("inf")
            for _ in range(3):
                s, e = rt.Event(), rt.Event()
                s.record()
                t0 = time.perf_counter()
                for _ in range(50):
                    fn(ov)
                host = (time.perf_counter() - t0) / 50
                e.record()
                e.synchronize()
                best = min(best, s.elapsed_ms(e) / 50)
            row[f"{name}{'_overlap' if ov else ''}_us"] = round(best * 1e3, 2)
            row[f"{name}{'_overlap' if ov else ''}_host_us"] = round(host * 1e6, 2)
    box.check()
    out[f"2^{lg}"] = row
    print(json.dumps({f"2^{lg}": row}), flush=True)
    for a in (x, y):
        a.free()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/probe_p2p_overhead.json").write_text(json.dumps(out, indent=1))
