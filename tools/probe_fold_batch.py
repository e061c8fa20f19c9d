"""Same-box A/B of the last CTA's partials fold, run while rtcg::finish
read each thread's run of partials through an out-of-line fold_range with
RTCG_FOLD_BATCH loads in flight: one dependent L2 load per partial
(RTCG_FOLD_BATCH=1) against batches of 16, for the 2^28 f32 dot
at the bench's tuned variants.  Both builds live in one process; the
measurements interleave (A, B, A, B, ...) so clocks and heat hit both alike.

  isolated_us   one launch between events, synchronised (median of 15)
  pdl_us        20 back-to-back overlapped launches / 20 (best of 3)

    python tools/probe_fold_batch.py > gpurun_out/probe_fold_batch.json

Result (profiles/r02_probe_fold_batch.json): level, -8 to +2 us per launch
by variant; the batched fold was reverted (the -D flag is now inert).
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, jit  # noqa: E402
from paper_0911_3456_b200 import ndarray as nd, reduction as rd  # noqa: E402


def main():
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    n = 1 << 28
    x, y = pool.alloc(nd.float32, (n,)), pool.alloc(nd.float32, (n,))
    rt.memset_async(x.address, 0x3c, n * 4)
    rt.memset_async(y.address, 0x3d, n * 4)
    o = pool.alloc(nd.float32, ())
    spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
    builds = {}
    for batch in (1, 16):
        cfg = jit.ToolchainConfig(flags=jit.DEFAULT_FLAGS + (f"-DRTCG_FOLD_BATCH={batch}",))
        for v in ((128, 1, 2), (256, 4, 2), (512, 1, 2), (1024, 1, 2)):
            builds[(batch, v)] = rd.ReductionKernel(
                spec, "dot_k", ew.VariantParams(block=v[0], unroll=v[1], waves=v[2]), config=cfg)
    rows = {f"{b}_{v[0]}_{v[1]}_{v[2]}": {"iso": [], "pdl": []} for b, v in builds}
    results = set()
    for _ in range(3):
        for (b, v), k in builds.items():
            row = rows[f"{b}_{v[0]}_{v[1]}_{v[2]}"]
            for _ in range(3):
                k.launch(x, y, out=o)
            rt.synchronize()
            for _ in range(5):
                s, e = rt.Event(), rt.Event()
                s.record()
                k.launch(x, y, out=o)
                e.record()
                e.synchronize()
                row["iso"].append(s.elapsed_ms(e) * 1e3)
            s, e = rt.Event(), rt.Event()
            s.record()
            for _ in range(20):
                k.launch(x, y, out=o, overlap_previous=True)
            e.record()
            e.synchronize()
            row["pdl"].append(s.elapsed_ms(e) * 1e3 / 20)
            results.add((v, float(o.get())))
    out = {key: {"isolated_us": round(statistics.median(r["iso"]), 1),
                 "pdl_us": round(min(r["pdl"]), 1)} for key, r in rows.items()}
    # the fold order is the same: every variant's result is identical across batches
    same = all(len({r for (vv, r) in results if vv == v}) == 1 for _, v in builds)
    print(json.dumps({"what": __doc__.split("\n\n")[0], "rows": out, "same_bits": same},
                     indent=1))


if __name__ == "__main__":
    main()
