"""Does the relative placement of the input streams matter?  dot / axpy at 2^28
f32 with y (and z) placed at byte offsets from a 1 GiB-aligned x."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402


def view(addr, n, dtype=nd.float32):
    a = object.__new__(nd.NdArray)

    class B:
        address = addr
    a.dtype, a.shape, a.size, a.nbytes = dtype, (n,), n, n * dtype.size
    a.pool, a._block, a._freed, a._finalizer = None, B, False, None
    return a


def dev_ms(fn, reps=40):
    fn()
    rt.synchronize()
    evs = [rt.Event() for _ in range(reps + 1)]
    evs[0].record()
    for j in range(reps):
        fn()
        evs[j + 1].record()
    evs[-1].synchronize()
    return evs[0].elapsed_ms(evs[-1]) / reps


rt.set_device(0)
N = 1 << 28
GB = 1 << 30
raw = rt.mem_alloc(3 * GB + (64 << 20))
base = (raw + GB - 1) // GB * GB if (raw + GB - 1) // GB * GB + 3 * GB <= raw + 3 * GB + (64 << 20) \
    else raw
rt.memset_async(raw, 0, 3 * GB + (64 << 20))
rt.synchronize()
print("raw", hex(raw), "base", hex(base), file=sys.stderr)
dot = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=8, block=256, waves=1))
axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                            "z[i] = a * x[i] + b * y[i]", "axpy",
                            ew.VariantParams(unroll=1, block=128, waves=0))
out = nd.MemoryPool(device=0).alloc_uninitialized(nd.float32, ())
rows = []
x = view(base, N)
for off in (0, 256, 512, 1024, 4096, 8192, 65536, 1 << 20, (1 << 20) + 256, 3 << 20,
            (7 << 20) + 4352, 16 << 20, 32 << 20):
    y = view(base + GB + off, N)
    ms = dev_ms(lambda: dot.launch(x, y, out=out))
    z = view(base + 2 * GB + 2 * off if 2 * off < (64 << 20) else base + 2 * GB + off, N)
    ms2 = dev_ms(lambda: axpy(2.0, x, -3.0, y, z))
    rows.append({"offset": off, "dot_GBs": round(8 * N / ms / 1e6), "axpy_GBs": round(12 * N / ms2 / 1e6)})
    print(json.dumps(rows[-1]))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/probe_offsets.json").write_text(json.dumps(rows, indent=1))
