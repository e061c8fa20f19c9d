"""Long stress of the in-kernel peer exchange: W emulated ranks on their own
streams, random per-rank delays, overlapped launches, many epochs, three
reduction kinds; every rank's result checked every epoch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import parallel as par, reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
world, epochs = 8, 400
x = rng.integers(-1000, 1000, 1_000_003).astype(np.int64)
bounds = [r * x.size // world for r in range(world + 1)]
shards = [(nd.from_host(pool, nd.int64, x[bounds[r]:bounds[r + 1]]), bounds[r])
          for r in range(world)]
# emulated ranks share the SMs: pin grids small and drain every 16 epochs so
# overlapped grids waiting on their predecessors can never fill the device
# (with one GPU per rank a waiting grid only waits on its own predecessor)
v = ew.VariantParams(workers=2)
kernels = [rd.sum_kernel(nd.int64, v), rd.max_kernel(nd.int64, v),
           rd.make_reduction("int64_t *x", nd.int64, "0", "a + b", "x[i] * x[i]", "sq", v)]
wants = [int(x.sum()), int(x.max()), int((x * x).sum())]
spin = ew.ElementwiseKernel("long iters, float *w", "float a = w[i]; for (long t = 0; "
                            "t < iters; ++t) a = a * 0.999f + 0.001f; w[i] = a", "spin")
busy = [pool.alloc(nd.float32, (2048,)) for _ in range(world)]
# load every module before any rank waits on the device: in one process a
# module load can wait for running kernels, i.e. for a rank spinning in its
# exchange (with one GPU per rank that is a stall, here it would deadlock)
spin(1, busy[0])
for k in kernels:
    k(shards[0][0])
rt.synchronize()
group = par.PeerMailbox.local_group(world)
streams = [rt.Stream() for _ in range(world)]
outs = [[pool.alloc_uninitialized(nd.int64, ()) for _ in range(world)] for _ in range(epochs)]
for j in range(epochs):
    k = kernels[j % 3]
    for r in rng.permutation(world):
        with rt.use_stream(streams[r].handle):
            if rng.random() < 0.5:
                spin(int(rng.integers(0, 30000)), busy[r])
            s = k.launch(shards[r][0], base=shards[r][1], peers=group[r],
                         overlap_previous=bool(rng.random() < 0.7))
            rt.memcpy_dtod(outs[j][r].address, s.result, 8)
    if j % 16 == 15:
        for st in streams:
            st.synchronize()
for st in streams:
    st.synchronize()
for m in group:
    m.check()
bad = [(j, r) for j in range(epochs) for r in range(world)
       if int(outs[j][r].get()[()]) != wants[j % 3]]
print(f"{epochs} epochs x {world} ranks: {len(bad)} wrong", bad[:5])
sys.exit(1 if bad else 0)
