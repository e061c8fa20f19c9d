"""Strong-scaling per-GPU shares on one B200: dot f32 at n = 2^25 / 2^26 /
2^27 (the 2^28-total workload split over 8 / 4 / 2 GPUs), tuned at that size
and at 2^28, timed as 50 back-to-back overlapped launches, local and with a
one-rank peer mailbox (the in-kernel exchange)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, autotune as at, elementwise as ew  # noqa: E402
from paper_0911_3456_b200 import ndarray as nd, parallel as par, reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
rng = np.random.default_rng(0)
X = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, 1 << 28).astype(np.float32))
Y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, 1 << 28).astype(np.float32))
o = pool.alloc_uninitialized(nd.float32, ())
box = par.PeerMailbox.local_group(1)[0]
axes = dict(at.DEFAULT_AXES, waves=(0, 1, 2), cache=("default", "tma"))
rows = {}
for lg in (25, 26, 27, 28):
    n = 1 << lg
    x, y = X[:n], Y[:n]
    t = at.tune_reduction(spec, "dot_k", n, axes, args=[x, y],
                          constraints=(lambda a: a["cache"] != "tma" or a["unroll"] == 1,),
                          protocol=at.MeasurementProtocol(warmup=1, repeats=3), burst=20)
    row = {}
    for label, v in (("tuned_here", t.best_assignment),
                     ("tuned_2p28", {"block": 256, "unroll": 1, "waves": 2})):
        k = rd.ReductionKernel(spec, "dot_k", ew.VariantParams(**v))
        for mode, fn in (("local", lambda: k.launch(x, y, out=o, overlap_previous=True)),
                         ("p2p", lambda: k.launch(x, y, out=o, peers=box,
                                                  overlap_previous=True))):
            timer = at.device_timer(fn, 50)
            timer()
            us = min(timer() for _ in range(3)) * 1e6
            row[f"{label}_{mode}_us"] = round(us, 2)
            row[f"{label}_{mode}_GBs"] = round(8 * n / us / 1e3, 1)
        row[f"{label}_variant"] = v
    rows[f"2^{lg}"] = row
    print(json.dumps({f"2^{lg}": row}), flush=True)
box.check()
Path("gpurun_out/probe_strong.json").write_text(json.dumps(rows, indent=1))
