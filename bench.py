"""Benchmark of the RTCG hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): ``ReductionKernel`` dot product
``sum(x*y)``, float32, n = 2^28 elements per GPU (weak scaling), block/unroll
autotuned before the timed region.  One step = one full reduction of the
resident inputs (per-CTA folds + in-kernel ordered combine; for N > 1 also the
NCCL all-gather of the per-rank partials and the rank-ordered combine).
``value`` = algorithmic bytes (8 B/element: x and y read once) of all ranks /
max-over-ranks device time.  Inputs (2 x 1 GiB per GPU) exceed the 126 MB L2,
so no flush is needed between steps.

The JSON line also carries: ``e2e`` (same metric through the public API with
pinned host inputs copied in and the scalar read back every step),
``roofline`` (dominant kernel vs MEASURED_PEAKS.json HBM copy bandwidth),
``cpu_baseline`` (the reference's CPU kernel on this host, bounded sample),
``clocks`` (NVML during the timed region) and ``workloads`` (the other
configs measured the same way: axpy, f64 poly+sin, max|x|, L2, int64 sum).

``--impl reference`` times the reference's own CPU implementation of the same
workload (``oracle/_ref``: C emitted by rtcg-kit's generator, compiled with its
command line, driven with its threading) on all host cores of rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_PER_GPU = 1 << 28
METRIC = "Elementwise/reduction GB/s vs B200 HBM peak at 1/2/4/8 GPU; speedup vs CPU ref"
WORKLOAD = "ReductionKernel dot sum(x*y) float32 n=2^28 per GPU, autotuned block/unroll"
FALLBACK_HBM = 6650.0
NOMINAL_HBM = 7672.0   # HBM3e spec: 3996 MHz x 2 transfers x 7680-bit bus / 8 (GB/s)


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        data = json.loads(path.read_text())
        return float(data["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


# --- clocks ------------------------------------------------------------------------------------


class ClockSampler:
    """NVML samples of SM clock and throttle reasons while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period: float = 0.02) -> None:
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # pragma: no cover - no NVML
            self._nv = None
            self.error = str(exc)

    def _sample(self):
        nv = self._nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for bit, name in self.REASONS.items():
            if mask & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self._period)

    def __enter__(self):
        if self._nv is not None:
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self._nv is not None:
            self._stop.set()
            self._t.join()
            self._sample()

    def summary(self) -> dict:
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.error}
        busy = [s for s in self.samples if s > 0]
        return {"sm_mhz": float(np.median(busy)) if busy else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons - {"gpu_idle"}),
                "samples": len(self.samples)}


# --- distributed plumbing ------------------------------------------------------------------------


class Dist:
    def __init__(self, gpus: int) -> None:
        self.world = _env_int("WORLD_SIZE", 1)
        self.rank = _env_int("RANK", 0)
        self.local = _env_int("LOCAL_RANK", 0)
        if self.world != gpus and "WORLD_SIZE" in os.environ:
            print(f"warning: --gpus {gpus} but WORLD_SIZE={self.world}", file=sys.stderr)
        self.torch = None
        # RTCG_BENCH_FORCE_DIST=1 runs the multi-GPU code path (process group,
        # cross-GPU exchange of the accumulators) even at world size 1
        self.forced = os.environ.get("RTCG_BENCH_FORCE_DIST") == "1"
        if self.world > 1 or self.forced:
            if "MASTER_ADDR" not in os.environ:
                import socket
                with socket.socket() as sock:
                    sock.bind(("127.0.0.1", 0))
                    port = sock.getsockname()[1]
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", str(port))
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.torch, self.dist = torch, dist

    @property
    def distributed(self) -> bool:
        return self.torch is not None

    def barrier(self):
        if self.distributed:
            self.dist.barrier()

    def max(self, value: float) -> float:
        if not self.distributed:
            return value
        t = self.torch.tensor([value], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.distributed:
            self.dist.destroy_process_group()


# --- CPU reference ---------------------------------------------------------------------------------


def cpu_reference(workload: str, steps: int | None = None, warmup: int = 1,
                  budget_s: float = 10.0, n_sample: int = 1 << 26):
    """Time the reference CPU kernel on a bounded sample of the workload.

    ``steps`` given: exactly that many timed calls after ``warmup`` (mean);
    else calls until ``budget_s`` (>= 3, <= 50; best).  Returns a dict."""
    from oracle import refdrive
    fn, kind = refdrive.load(workload)
    threads = refdrive.host_threads()
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, n_sample).astype(np.float32)
    y = rng.uniform(-1, 1, n_sample).astype(np.float32)
    for _ in range(max(1, warmup)):
        fn(x, y, workers=threads)  # page in, thread spin-up
    times = []
    if steps is not None:
        t0 = time.perf_counter()
        for _ in range(steps):
            fn(x, y, workers=threads)
        per_call, stat = (time.perf_counter() - t0) / steps, f"mean of {steps} calls"
    else:
        t_end = time.perf_counter() + budget_s
        while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 50):
            t0 = time.perf_counter()
            fn(x, y, workers=threads)
            times.append(time.perf_counter() - t0)
        per_call, stat = min(times), f"best of {len(times)} calls"
    return {"value": round(8 * n_sample / per_call / 1e9, 3), "unit": "GB/s", "cores": threads,
            "kind": kind, "seconds_per_call": per_call,
            "calls": steps if steps is not None else len(times),
            "sample": f"dot f32 n=2^{int(math.log2(n_sample))} per call (bounded sample of the "
                      f"2^28 workload), x,y~U(-1,1) seed 0, reference variant unroll=4 "
                      f"contiguous-blocks, {threads} worker threads, {stat}"}


def run_reference(args) -> int:
    """CPU reference arm: rank 0 only, no GPU or process group needed."""
    if _env_int("RANK", 0) != 0:
        return 0
    base = cpu_reference("dot_k", steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(base["seconds_per_call"] * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": WORKLOAD + " (CPU: bounded sample)",
                                            "n": 1 << 26},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# --- GPU arm ----------------------------------------------------------------------------------------


def _time_steps(rt, step, k: int, per_step: bool = True):
    """Device time of k steps on the current stream, plus per-step durations
    (``per_step=False``: only the two bracketing events, so nothing is
    recorded between back-to-back launches; per-step = the mean)."""
    if not per_step:
        start, stop = rt.Event(), rt.Event()
        start.record()
        for _ in range(k):
            step()
        stop.record()
        stop.synchronize()
        total = start.elapsed_ms(stop)
        return total, [total / k] * k
    events = [rt.Event() for _ in range(k + 1)]
    events[0].record()
    for j in range(k):
        step()
        events[j + 1].record()
    events[-1].synchronize()
    per = [events[j].elapsed_ms(events[j + 1]) for j in range(k)]
    return events[0].elapsed_ms(events[-1]), per


def run_ours(args) -> int:
    d = Dist(args.gpus)
    from paper_0911_3456_b200 import _runtime as rt
    from paper_0911_3456_b200 import autotune as at
    from paper_0911_3456_b200 import ndarray as nd
    from paper_0911_3456_b200 import parallel as par
    from paper_0911_3456_b200 import reduction as rd
    from paper_0911_3456_b200 import elementwise as ew

    rt.set_device(d.local)
    info = rt.device_info(d.local)
    stream_handle = d.torch.cuda.current_stream().cuda_stream if d.distributed else 0
    pool = nd.MemoryPool(device=d.local)
    n = N_PER_GPU
    total_n = n * d.world
    peak, peak_kind = _peaks()

    with rt.use_stream(stream_handle):
        # resident inputs: this rank's slice of a global 2^28*N array
        lo, _ = par.shard_range(total_n, d.rank, d.world)
        hx = nd.pinned_empty((n,), nd.float32)
        hy = nd.pinned_empty((n,), nd.float32)
        rng = np.random.default_rng([0, d.rank])
        hx[:] = rng.uniform(-1, 1, n).astype(np.float32)
        hy[:] = rng.uniform(-1, 1, n).astype(np.float32)
        gx, gy = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
        sx = par.ShardedArray(gx, lo, total_n, d.rank, d.world)
        sy = par.ShardedArray(gy, lo, total_n, d.rank, d.world)

        # autotune block x unroll for (dot, float32, n) -- outside the timed region
        spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
        t0 = time.perf_counter()
        # variants ranked as the metric is measured: mean of back-to-back launches
        axes = dict(at.DEFAULT_AXES, waves=(0, 1, 2), cache=("default", "tma"))
        tuned = at.tune_reduction(spec, "dot_k", n, axes, args=[gx, gy],
                                  constraints=(lambda a: a["cache"] != "tma" or a["unroll"] == 1,),
                                  protocol=at.MeasurementProtocol(warmup=1, repeats=3),
                                  store=at.TuneStore(), burst=10)
        out = pool.alloc_uninitialized(nd.float32, ())
        # confirmation stage: the tuner's top 8 re-timed over 50-launch bursts of
        # overlapped launches (how the timed steps run)
        # (its 3 x 10-launch samples leave ~1-2 % of noise in the ranking)
        finalists = sorted((e for e in tuned.table if e.status == "ok"),
                           key=lambda e: e.stat_seconds)[:8]
        confirm = []
        for e in finalists:
            k = rd.ReductionKernel(spec, "dot_k", ew.VariantParams(**e.as_dict()))
            run = at.device_timer(lambda k=k: k.launch(gx, gy, out=out,
                                                       overlap_previous=True), 50)
            run()
            confirm.append((min(run() for _ in range(2)), e.as_dict()))
        best = min(confirm, key=lambda c: c[0])[1] if confirm else tuned.best_assignment
        if os.environ.get("RTCG_BENCH_DOT_VARIANT"):   # experiments: pin the variant
            best = json.loads(os.environ["RTCG_BENCH_DOT_VARIANT"])
        tune_s = time.perf_counter() - t0
        kernel = rd.ReductionKernel(spec, "dot_k", ew.VariantParams(**best))

        collective = None
        # steps are back-to-back reductions over inputs nothing writes, so each
        # may start streaming while the previous one folds (programmatic
        # dependent launch; ReductionKernel.launch(overlap_previous=True))
        if not d.distributed:
            def step():
                kernel.launch(gx, gy, out=out, overlap_previous=True)
        else:
            # the product path: one launch per GPU, accumulators exchanged over
            # NVLink peer memory inside the kernel; NCCL only when peers are
            # unreachable (RTCG_BENCH_COLLECTIVE overrides, e.g. "allgather")
            collective = os.environ.get("RTCG_BENCH_COLLECTIVE") or (
                "p2p" if par.p2p_capable() else "auto")

            def step():
                par.sharded_reduce(kernel, sx, sy, return_device=True, collective=collective,
                                   overlap_previous=collective == "p2p").free()

        # correctness of the tuned kernel on this data (cheap, before timing)
        value = kernel(gx, gy)
        terms_ok = bool(np.isfinite(value))
        # the tuned kernel against an fp64 oracle on the same data: products
        # rounded in float32 (C semantics), summed in float64 by numpy
        terms = np.multiply(hx, hy, dtype=np.float32).astype(np.float64)
        want = float(np.sum(terms))
        bound = 0.5 * float(np.spacing(np.float32(abs(want)))) + \
            2 * n * 2.0**-53 * float(np.abs(terms).sum())
        check = {"got": float(value), "want_fp64": want, "bound": bound,
                 "ulps_f32": abs(float(value) - want) / float(np.spacing(np.float32(abs(want)))),
                 "ok": abs(float(value) - want) <= bound}
        del terms

        try:
            step()
            if collective == "p2p":   # every rank must agree the exchange works
                timed_out = 0.0
                try:
                    par.peer_mailbox(None, stream_handle).check(stream_handle)
                except par.PeerTimeout:
                    timed_out = 1.0
                if d.max(timed_out) > 0:
                    raise RuntimeError("the peer exchange timed out on some rank")
        except Exception as exc:  # p2p refused or broken here: the NCCL baseline
            if collective != "p2p":
                raise
            print(f"warning: p2p exchange unavailable ({exc}); using NCCL", file=sys.stderr)
            collective = "auto"
            step()
        for _ in range(max(3, args.warmup)):
            step()
        rt.synchronize()
        d.barrier()
        rt.synchronize()
        launches0 = kernel.launches
        with ClockSampler(d.local) as clocks:
            total_ms, per_step = _time_steps(rt, step, args.steps,
                                             os.environ.get("RTCG_BENCH_STEP_EVENTS", "0") == "1")
        # NCCL paths add one combine launch per step; p2p is one kernel
        launches = kernel.launches - launches0 + (
            args.steps if d.distributed and collective != "p2p" else 0)
        rt.synchronize()
        d.barrier()
        step_ms = d.max(total_ms / args.steps)
        kern_ms = float(np.mean(per_step))
        value_gbs = 8 * total_n / (step_ms * 1e-3) / 1e9

        # e2e through the public API: pinned host -> device, reduce, scalar back
        e2e_steps = max(2, min(args.steps, 5))
        h2d = 2 * n * 4
        gx2, gy2 = pool.alloc_uninitialized(nd.float32, (n,)), pool.alloc_uninitialized(nd.float32, (n,))

        from paper_0911_3456_b200 import driver as drv
        sx2 = par.ShardedArray(gx2, lo, total_n, d.rank, d.world)
        sy2 = par.ShardedArray(gy2, lo, total_n, d.rank, d.world)

        def e2e_sequential():
            gx2.copy_from_host(hx, sync=False)
            gy2.copy_from_host(hy, sync=False)
            if d.distributed:           # this rank's slice, then the cross-GPU combine
                return par.sharded_reduce(kernel, sx2, sy2, collective=collective)
            return kernel(gx2, gy2)     # returns the host scalar (4-byte DtoH)

        def e2e_streamed():             # dot(driver.In(x), driver.In(y)): chunked, overlapped
            return kernel(drv.In(hx), drv.In(hy))

        def time_e2e(fn):
            fn()
            d.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                fn()
            return d.max((time.perf_counter() - t0) / e2e_steps)
        # copy-in then reduce: the inputs cross the link once, whole (the
        # measured best for a one-way workload; the streamed host call adds
        # per-chunk overhead and is reported beside it at N = 1)
        e2e_s = time_e2e(e2e_sequential)
        streamed_s = None if d.distributed else time_e2e(e2e_streamed)
        e2e_gbs = 8 * total_n / e2e_s / 1e9
        # the link roofline for e2e: raw pinned HtoD copy of the same bytes
        t0 = time.perf_counter()
        for _ in range(2):
            gx2.copy_from_host(hx, sync=False)
            gy2.copy_from_host(hy, sync=True)
        link_gbs = 2 * h2d / (time.perf_counter() - t0) / 1e9
        gx2.free()
        gy2.free()

        workloads = {} if args.quick or d.world > 1 else \
            secondary_workloads(rt, nd, ew, rd, at, pool, peak)

    algo_bytes = 8 * n
    achieved = algo_bytes / (kern_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value_gbs, 2), "unit": "GB/s", "n_gpus": d.world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(step_ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_per_gpu": n, "n_total": total_n,
                   "variant": best, "autotune_seconds": round(tune_s, 2),
                   "autotune_from_store": tuned.from_store,
                   "l2": "inputs 2 GiB per GPU > 126 MB L2 (no flush needed)",
                   "parallelism": f"shards{d.world}" + (f"+{collective}" if d.distributed
                                                        else ""),
                   "accumulator": "float64",
                   "launch": "back-to-back steps with programmatic dependent launch (each "
                             "reduction streams its inputs while the previous one folds)",
                   "gpu": info["name"], "result_finite": terms_ok,
                   "result_vs_fp64_oracle": check},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy)"
                     if peak_kind == "measured" else "fallback (B200_PROFILING.md)",
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "nominal_peak": NOMINAL_HBM,
                     "frac_of_nominal": round(achieved / NOMINAL_HBM, 4),
                     "traffic": _ncu_traffic("dot_k"),
                     "kernel": kernel.launch_config(gx, gy)["entry"],
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "avg_kernel_ms": round(kern_ms, 4)},
        "e2e": {"value": round(e2e_gbs, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4, "steps": e2e_steps,
                "path": "GPUArray.copy_from_host (pinned) x2 + "
                        + ("sharded_reduce" if d.distributed else "ReductionKernel.__call__")
                        + " (numpy scalar)",
                "streamed_value": None if streamed_s is None else
                round(8 * total_n / streamed_s / 1e9, 2),
                "streamed_path": "ReductionKernel(driver.In(x), driver.In(y)): 64 MiB chunks, "
                                 "uploads overlapped with per-chunk reductions",
                "link_h2d_gbs": round(link_gbs, 2),
                "link_frac": round(e2e_gbs / (link_gbs * d.world), 4),
                "note": "every input byte crosses the host link once per step, so e2e is "
                        "bounded by the measured pinned HtoD bandwidth (link_h2d_gbs)"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "workloads": workloads,
    }
    if d.world == 1 and d.rank == 0 and not args.no_cpu:
        try:
            base = cpu_reference("dot_k", budget_s=10.0)
            line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind",
                                                         "sample")}
        except Exception as exc:  # pragma: no cover - report, don't fail the bench
            line["cpu_baseline"] = {"value": None, "error": str(exc)}
    if d.rank == 0:
        emit(line)
    d.close()
    return 0


def _ncu_traffic(kernel: str):
    """dram bytes per launch from the committed ncu summary, if captured."""
    path = ROOT / "profiles" / "ncu_summary.json"
    try:
        data = json.loads(path.read_text())
        return data["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def secondary_workloads(rt, nd, ew, rd, at, pool, peak):
    """The other BASELINE configs on one GPU: each kernel autotuned over
    unroll x block (TuneStore-cached), then device-timed (best of 10)."""
    out = {}
    n = N_PER_GPU
    rng = np.random.default_rng(1)
    proto = at.MeasurementProtocol(warmup=1, repeats=3)
    store = at.TuneStore()

    def best_ms(fn, reps=5, burst=10):
        """Per-launch time as the headline measures it: the mean of a burst of
        back-to-back launches between two events (best of ``reps`` bursts)."""
        fn()
        rt.synchronize()
        best = math.inf
        for _ in range(reps):
            ms, _ = _time_steps(rt, fn, burst, per_step=False)
            best = min(best, ms / burst)
        return best

    def record(name, fn, nbytes, tuned, **extra):
        with ClockSampler(rt.current_device()) as clk:
            ms = best_ms(fn)
        extra = dict(extra, clocks=clk.summary())
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4),
                     "algorithmic_bytes": nbytes, "variant": tuned.best_assignment,
                     "tune_from_store": tuned.from_store, **extra}

    x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    z = pool.alloc_uninitialized(nd.float32, (n,))
    sig, op = "float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]"
    axes = dict(at.DEFAULT_AXES, waves=(0, 1, 2))
    t = at.tune_elementwise(sig, op, "axpy", n, axes, args=[2.0, x, -3.0, y, z],
                            protocol=proto, store=store, burst=10)
    axpy = ew.ElementwiseKernel(sig, op, "axpy", ew.VariantParams(**t.best_assignment))
    record("axpy_f32_2p28", lambda: axpy(2.0, x, -3.0, y, z), 12 * n, t)
    for a in (x, y, z):
        a.free()

    # C4: max|x|, L2 (sum of squares; sqrt on the host) and the wrapping int64
    # sum at n = 2^32, inputs synthesised on the device from a hash of i
    big = 1 << 32
    xf = pool.alloc_uninitialized(nd.float32, (big,))
    ew.ElementwiseKernel("float *x", "unsigned long h = (unsigned long) i * 0x9E3779B97F4A7C15UL; "
                         "x[i] = (float) ((long) (h >> 40) - (1L << 23)) * 1.1920929e-7f",
                         "synth_f32")(xf)
    o32 = pool.alloc_uninitialized(nd.float32, ())
    for name, mp, red in (("maxabs", "fabsf(x[i])", "a > b ? a : b"),
                          ("sumsq", "x[i] * x[i]", "a + b")):
        spec = rd.ReductionSpec("float *x", nd.float32, "0", red, mp)
        t = at.tune_reduction(spec, name, big, axes, args=[xf], protocol=proto,
                              store=store, burst=3)
        k = rd.ReductionKernel(spec, name, ew.VariantParams(**t.best_assignment))
        record(f"{name}_f32_2p32", lambda: k.launch(xf, out=o32, overlap_previous=True),
               4 * big, t,
               note="L2 norm = sqrt(sumsq) on the host" if name == "sumsq" else "max|x|")
    xf.free()
    xi = pool.alloc_uninitialized(nd.int64, (big,))
    ew.ElementwiseKernel("long *x", "x[i] = (long) ((unsigned long) i * 0x9E3779B97F4A7C15UL) >> 1",
                         "synth_i64")(xi)
    o64 = pool.alloc_uninitialized(nd.int64, ())
    spec = rd.ReductionSpec("int64_t *x", nd.int64, "0", "a + b")
    t = at.tune_reduction(spec, "sum_k", big, axes, args=[xi], protocol=proto,
                          store=store, burst=3)
    si = rd.ReductionKernel(spec, "sum_k", ew.VariantParams(**t.best_assignment))
    record("sum_i64_2p32", lambda: si.launch(xi, out=o64, overlap_previous=True), 8 * big, t,
           note="values in [-2^62, 2^62): the sum wraps (bit-exact, order independent)")
    xi.free()

    hx = nd.pinned_empty((n,), nd.float64)
    hx[:] = rng.uniform(-2, 2, n)
    xd = nd.from_host(pool, nd.float64, hx)
    zd = pool.alloc_uninitialized(nd.float64, (n,))
    sig, op = ("double a, double *x, double *z",
               "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])")
    # long statements: the software-pipelined loop keeps loads in flight
    ps_axes = dict(axes, waves=(0, 1, 2, 4), prefetch=(False, True))
    t = at.tune_elementwise(sig, op, "polysin", n, ps_axes, args=[0.5, xd, zd],
                            constraints=(lambda a: not a["prefetch"] or a["waves"] > 0,),
                            protocol=proto, store=store, burst=10)
    ps = ew.ElementwiseKernel(sig, op, "polysin", ew.VariantParams(**t.best_assignment))
    record("polysin_f64_2p28", lambda: ps(0.5, xd, zd), 16 * n, t,
           bound="instruction issue + HBM: ~67 instructions/element (~21 FP64); ncu: issue "
                 "slots 68% busy, FP64 pipe 44%, DRAM 68.5% (profiles/r01_ncu_full_polysin_*); "
                 "the prefetch variant keeps the next chunk's loads in flight")
    # C3 end to end through the public API: pinned host x -> HBM, kernel, HBM ->
    # pinned host z (16 B/element cross the host link), against the reference's
    # CPU kernel on all host cores -- the compute-heavy case where the GPU wins
    # end to end even though every byte crosses PCIe.
    hz = nd.pinned_empty((n,), nd.float64)
    from paper_0911_3456_b200 import driver as drv

    def e2e_sequential():
        xd.copy_from_host(hx, sync=False)
        ps(0.5, xd, zd)
        zd.to_host(out=hz)

    def e2e_streamed():           # chunked upload / kernel / download on two streams
        ps(0.5, drv.In(hx), drv.Out(hz))

    def timed(fn, reps=3):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps
    seq_s, str_s = timed(e2e_sequential), timed(e2e_streamed)
    out["polysin_f64_2p28"]["e2e"] = {
        "value": round(16 * n / str_s / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": 8 * n,
        "d2h_bytes_per_step": 8 * n, "steps": 3,
        "path": "ElementwiseKernel(0.5, driver.In(x), driver.Out(z)) on pinned host arrays: "
                "64 MiB chunks, upload / kernel / download overlapped on two streams",
        "sequential_value": round(16 * n / seq_s / 1e9, 2),
        "sequential_path": "GPUArray.copy_from_host + ElementwiseKernel + GPUArray.to_host"}
    try:
        from oracle import refdrive
        fn, kind = refdrive.load("polysin")
        threads = refdrive.host_threads()
        m = 1 << 23
        cx, cz = np.ascontiguousarray(hx[:m]), np.empty(m)
        fn(0.5, cx, cz, workers=threads)
        best = math.inf
        for _ in range(5):
            t0 = time.perf_counter()
            fn(0.5, cx, cz, workers=threads)
            best = min(best, time.perf_counter() - t0)
        out["polysin_f64_2p28"]["cpu_baseline"] = {
            "value": round(16 * m / best / 1e9, 3), "unit": "GB/s", "cores": threads,
            "kind": kind, "sample": f"polysin f64 n=2^23 (bounded sample), x~U(-2,2), "
                                    f"reference variant, {threads} worker threads, best of 5"}
    except Exception as exc:  # pragma: no cover - report, don't fail the bench
        out["polysin_f64_2p28"]["cpu_baseline"] = {"value": None, "error": str(exc)}
    xd.free()
    zd.free()
    return out


_JSON_OUT = None


def emit(line: dict) -> None:
    """Write the one JSON result line to the real stdout (native libraries --
    NCCL's version banner, for one -- were redirected to stderr)."""
    text = json.dumps(line) + "\n"
    if _JSON_OUT is None:
        sys.stdout.write(text)
        sys.stdout.flush()
    else:
        os.write(_JSON_OUT, text.encode())


def _isolate_stdout() -> None:
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.dup(1)
    os.dup2(2, 1)


def main(argv=None) -> int:
    p = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--quick", action="store_true", help="skip the secondary workloads")
    p.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    args = p.parse_args(argv)
    _isolate_stdout()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    raise SystemExit(main())
