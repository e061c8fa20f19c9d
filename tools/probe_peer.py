"""Debug the emulated-rank exchange: one case per process (argv[1])."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, parallel as par  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
case = sys.argv[1]
x = np.random.default_rng(9).integers(-(1 << 62), 1 << 62, 1_000_003, dtype=np.int64)
if case == "i64_nonempty":
    parts, bases = [x[:600_000], x[600_000:]], (0, 600_000)
elif case == "i64_empty_middle":
    parts, bases = [x[:600_000], x[600_000:600_000], x[600_000:]], (0, 600_000, 600_000)
elif case == "i64_single_empty":
    parts, bases = [x[:0]], (0,)
else:
    parts, bases = [x[:600_000], x[600_000:700_000], x[700_000:]], (0, 600_000, 700_000)
shards = [([nd.from_host(pool, nd.int64, p)], b) for p, b in zip(parts, bases)]
group = par.PeerMailbox.local_group(len(parts))
k = rd.sum_kernel(nd.int64)
streams = [rt.Stream() for _ in parts]
t0 = time.time()
for r, ((args, base), st) in enumerate(zip(shards, streams)):
    with rt.use_stream(st.handle):
        print("rank", r, k.launch_config(*args) if args[0].size else "empty", flush=True)
        k.launch(*args, base=base, peers=group[r])
for st in streams:
    st.synchronize()
print(case, "ok", time.time() - t0, [int(k._read(k.scratch(0, st.handle).result, nd.int64))
                                    for st in streams], int(x.sum()), flush=True)
