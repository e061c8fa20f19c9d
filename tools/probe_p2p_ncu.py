"""ncu probe of the peer exchange's device cost at world size 1: dot f32
launches local vs with a one-rank mailbox (run under ncu -k regex:dot_p;
profiles/r02_probe_p2p_ncu.json holds the protocol history)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, jit, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import parallel as par, reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
for lg in (20, 28):
    n = 1 << lg
    x = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    y = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    o = pool.alloc_uninitialized(nd.float32, ())
    for proto in (0,):
        cfg = jit.ToolchainConfig()
        k = rd.ReductionKernel(rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b",
                                                "x[i] * y[i]"), f"dot_p{proto}",
                               ew.VariantParams(block=256, unroll=1, waves=2), config=cfg)
        box = par.PeerMailbox.local_group(1)[0]
        for _ in range(3):
            k.launch(x, y, out=o)
            k.launch(x, y, out=o, peers=box)
        rt.synchronize()
        assert float(o.get()[()]) == n
        box.check()
