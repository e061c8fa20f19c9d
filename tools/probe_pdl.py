"""Programmatic dependent launch for back-to-back reductions: dot f32 at 2^24,
2^26, 2^28 launched 200x plain vs with overlap_previous=True (the next
launch streams its inputs while the previous one folds); results checked."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402


def mean_ms(fn, reps=200):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_ms(e) / reps


rt.set_device(0)
pool = nd.MemoryPool(device=0)
rng = np.random.default_rng(0)
for lg in (20, 24, 26, 28):
    n = 1 << lg
    x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    o = pool.alloc_uninitialized(nd.float32, ())
    k = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=1, block=256, waves=1))
    want = float(k(x, y))
    plain = mean_ms(lambda: k.launch(x, y, out=o))
    over = mean_ms(lambda: k.launch(x, y, out=o, overlap_previous=True))
    got = float(o.get())
    print(f"2^{lg}: plain {plain * 1e3:.1f} us ({8 * n / plain / 1e6:.0f} GB/s)  overlapped "
          f"{over * 1e3:.1f} us ({8 * n / over / 1e6:.0f} GB/s)  result ok {got == want}",
          flush=True)
    for a in (x, y, o):
        a.free()
