"""Tuner semantics with an injected clock (reference tests/test_autotune.py and
acceptance test_06) plus device-timed tuning on the GPU (acceptance test_07)."""

import math

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_0911_3456_b200 import autotune as at
from paper_0911_3456_b200 import jit

GRID = {"unroll": (1, 2, 4, 8), "block": (128, 256, 512)}
PROTO = at.MeasurementProtocol(warmup=1, repeats=3, statistic="minimum", timeout_seconds=1e9)


class FakeClock:
    def __init__(self):
        self.now = 0.0

    def __call__(self):
        return self.now

    def runnable(self, cost):
        def run():
            self.now += cost
        return run


def oracle_factory(clock, cost_of):
    return lambda a: clock.runnable(cost_of(a))


@pytest.fixture(scope="module")
def fp():
    return jit.PlatformFingerprint(os="test-os", cpu="test-cpu", cores=1,
                                   toolchain="test-nvrtc 1.0", toolkit_version="0.1.0")


def test_enumeration():
    assert len(at.ParamSpace.make(GRID).enumerate()) == 12
    c = at.ParamSpace.make(GRID, constraints=(lambda a: a["unroll"] * a["block"] <= 2048,))
    got = c.enumerate()
    assert len(got) == 11 and {"unroll": 8, "block": 512} not in got
    assert at.ParamSpace.make({"unroll": (1,)}).enumerate() == [{"unroll": 1}]
    assert at.ParamSpace.make({"workers": (1, 2), "unroll": (4, 1)}).enumerate() == [
        {"unroll": 4, "workers": 1}, {"unroll": 4, "workers": 2},
        {"unroll": 1, "workers": 1}, {"unroll": 1, "workers": 2}]
    with pytest.raises(at.EmptySpace):
        at.ParamSpace.make({"u": (1, 2)}, constraints=(lambda a: False,)).enumerate()
    with pytest.raises(at.EmptySpace):
        at.ParamSpace.make({}).enumerate()


@given(st.dictionaries(st.sampled_from(["p", "q", "r"]),
                       st.lists(st.integers(0, 9), min_size=1, max_size=4, unique=True),
                       min_size=1, max_size=3))
def test_enumerate_count_is_product(axes):
    assert len(at.ParamSpace.make(axes).enumerate()) == math.prod(len(v) for v in axes.values())


def test_measure_protocol():
    clock = FakeClock()
    calls = []

    def run():
        calls.append(1)
        clock.now += 1e-3
    m = at.measure(run, at.MeasurementProtocol(warmup=2, repeats=3), clock=clock)
    assert len(calls) == 5 and len(m.samples) == 3
    for stat, want in (("median", 4e-3), ("minimum", 3e-3)):
        deltas = iter([5e-3, 3e-3, 4e-3])
        m = at.measure(lambda: setattr(clock, "now", clock.now + next(deltas)),
                       at.MeasurementProtocol(warmup=0, repeats=3, statistic=stat,
                                              timeout_seconds=1e9), clock=clock)
        assert m.seconds == pytest.approx(want)
    with pytest.raises(at.VariantTimeout):
        at.measure(clock.runnable(0.7), at.MeasurementProtocol(warmup=0, repeats=3,
                                                               timeout_seconds=1.0), clock=clock)
    with pytest.raises(at.VariantCrashed) as err:
        at.measure(lambda: 1 / 0, PROTO, clock=FakeClock())
    assert "ZeroDivisionError" in str(err.value)


def test_measure_prefers_self_reported_device_time():
    clock = FakeClock()
    m = at.measure(lambda: (setattr(clock, "now", clock.now + 1.0), 2e-6)[1], PROTO, clock=clock)
    assert m.seconds == 2e-6


def test_protocol_validation():
    for bad in (dict(repeats=0), dict(warmup=-1), dict(statistic="mean"),
                dict(timeout_seconds=0)):
        with pytest.raises(ValueError):
            at.MeasurementProtocol(**bad)


def test_tune_argmin_ties_and_determinism(fp):
    clock = FakeClock()
    space = at.ParamSpace.make(GRID)
    r = at.tune(oracle_factory(clock, lambda a: (10 - a["unroll"]) * 1e-3 + a["block"] * 1e-7),
                space, PROTO, fp=fp, clock=clock, prune=False)
    assert r.best_assignment == {"unroll": 8, "block": 128}
    r = at.tune(oracle_factory(clock, lambda a: 1e-3), space, PROTO, fp=fp, clock=clock,
                prune=False)
    assert r.best_assignment == {"block": 128, "unroll": 1}
    runs = [at.tune(oracle_factory(FakeClock(), lambda a: a["block"] * 1e-6), space, PROTO,
                    fp=fp, clock=FakeClock()) for _ in range(2)]
    assert runs[0] == runs[1]


def test_tune_isolates_failures(fp):
    clock = FakeClock()

    def factory(a):
        if a["unroll"] == 2:
            return lambda: 1 / 0
        if a == {"unroll": 1, "block": 128}:
            raise OSError("compile failed")
        return clock.runnable(a["unroll"] * 1e-3)
    r = at.tune(factory, at.ParamSpace.make(GRID), PROTO, fp=fp, clock=clock, prune=False)
    crashed = [e for e in r.table if e.status == "crashed"]
    assert len(crashed) == 4 and "compile failed" in r.table[0].reason
    assert r.best_assignment["unroll"] == 1 and r.best_assignment["block"] != 128
    with pytest.raises(at.AllVariantsFailed) as err:
        at.tune(lambda a: (_ for _ in ()).throw(RuntimeError("x")), at.ParamSpace.make(GRID),
                PROTO, fp=fp, clock=FakeClock())
    assert len(err.value.reasons) == 12 and "block=512,unroll=8" in err.value.reasons


def test_tune_timeouts(fp):
    clock = FakeClock()
    proto = at.MeasurementProtocol(warmup=0, repeats=2, timeout_seconds=0.1)
    r = at.tune(oracle_factory(clock, lambda a: 1.0 if a["block"] == 512 else 1e-3),
                at.ParamSpace.make(GRID), proto, fp=fp, clock=clock, prune=False)
    assert sum(e.status == "timeout" for e in r.table) == 4
    assert r.best_assignment["block"] != 512


def test_prune(fp):
    clock = FakeClock()
    r = at.tune(oracle_factory(clock, lambda a: 1e-2 if a["block"] == 512 else 1e-3),
                at.ParamSpace.make(GRID), PROTO, fp=fp, clock=clock, prune=True)
    pruned = [dict(e.assignment) for e in r.table if e.status == "pruned"]
    assert pruned and all(p["block"] == 512 for p in pruned)
    r = at.tune(oracle_factory(clock, lambda a: 1e-3 + a["unroll"] * 1e-4),
                at.ParamSpace.make(GRID), PROTO, fp=fp, clock=clock, prune=True)
    assert all(e.status == "ok" for e in r.table)


@given(st.lists(st.integers(1, 40), min_size=4, max_size=4))
def test_prune_exact_when_cost_depends_on_one_axis(costs):
    fp = jit.PlatformFingerprint(os="t", cpu="t", cores=1, toolchain="t", toolkit_version="0")
    per = dict(zip((1, 2, 4, 8), costs))
    clock = FakeClock()
    r = at.tune(oracle_factory(clock, lambda a: per[a["unroll"]] * 1e-3),
                at.ParamSpace.make(GRID), PROTO, fp=fp, clock=clock, prune=True)
    assert per[r.best_assignment["unroll"]] == min(per.values())


def test_sampling(fp):
    clock = FakeClock()
    space = at.ParamSpace.make(GRID)
    f = oracle_factory(clock, lambda a: 1e-3)
    r1 = at.tune(f, space, PROTO, fp=fp, clock=clock, sample=5, seed=3, prune=False)
    r2 = at.tune(f, space, PROTO, fp=fp, clock=clock, sample=5, seed=3, prune=False)
    ok1 = [e.assignment for e in r1.table if e.status == "ok"]
    assert len(ok1) == 5 and ok1 == [e.assignment for e in r2.table if e.status == "ok"]
    assert sum(e.status == "unsampled" for e in r1.table) == 7


def test_store_round_trip_warm_hit_and_layout(tmp_path, fp):
    store = at.TuneStore(tmp_path)
    clock = FakeClock()
    builds = []

    def factory(a):
        builds.append(a)
        return clock.runnable(a["unroll"] * 1e-3)
    space = at.ParamSpace.make(GRID)
    cold = at.tune(factory, space, PROTO, store=store, problem_key="dot/f32/2^28", fp=fp,
                   clock=clock)
    n_builds = len(builds)
    warm = at.tune(factory, space, PROTO, store=store, problem_key="dot/f32/2^28", fp=fp,
                   clock=clock)
    assert len(builds) == n_builds and warm.from_store and not cold.from_store
    assert warm == cold and warm.best_seconds == cold.best_seconds
    assert at.TuneResult.from_json(cold.to_json()) == cold
    other = jit.PlatformFingerprint(os="test-os", cpu="test-cpu", cores=1,
                                    toolchain="upgraded 2.0", toolkit_version="0.1.0")
    assert store.load(other, "dot/f32/2^28") is None
    path = store._path(fp, "junk")
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text("{broken")
    assert store.load(fp, "junk") is None
    at.tune(factory, space, PROTO, store=store, problem_key="probe", fp=fp, clock=clock)
    assert (tmp_path / "tune" / fp.digest() / "probe.json").exists()
    with pytest.raises(ValueError):
        at.tune(factory, space, PROTO, store=store, fp=fp, clock=clock)


def test_axes_are_validated():
    with pytest.raises(ValueError):
        at._check_axes({"threads": (1,)})
    assert at._check_axes(None) == at.DEFAULT_AXES
    # every VariantParams field is a tunable axis, dynamic chunks included
    assert at._check_axes({"chunk": (0, 8192), "waves": (1,)})["chunk"] == (0, 8192)
    from paper_0911_3456_b200 import elementwise as ew
    with pytest.raises(ValueError):
        ew.VariantParams(chunk=1000)                   # not a candidate size
    with pytest.raises(ValueError):
        ew.VariantParams(chunk=8192, cache="tma")      # the LDG vector path only
    sig = ew.parse_signature("float *x, float *z")
    with pytest.raises(ValueError):                    # reductions only
        ew.generate(sig, "z[i] = x[i]", "k", ew.VariantParams(chunk=8192))


# --- real kernels on the GPU -------------------------------------------------------------------


@pytest.mark.gpu
def test_tuned_axpy_is_near_best_and_beats_worst(pool, shared_cache):
    """Acceptance test_07 on the device: the tuned variant re-measures within
    1.25x of the best and faster than the worst."""
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd
    n = 1 << 24
    rng = np.random.default_rng(3)
    x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
    z = pool.alloc(nd.float32, (n,))
    sig, op = "float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]"
    axes = {"unroll": (1, 4), "block": (32, 256), "workers": (4, None)}
    proto = at.MeasurementProtocol(warmup=2, repeats=7)
    result = at.tune_elementwise(sig, op, "lincomb_tuned", n, axes, args=[2.0, x, -3.0, y, z],
                                 protocol=proto, cache=shared_cache, prune=False)

    def time_of(a):
        k = ew.make_elementwise(sig, op, "lincomb_tuned", ew.VariantParams(**a),
                                cache=shared_cache)
        return at.measure(at.device_timer(lambda: k(2.0, x, -3.0, y, z, n=n)), proto).seconds
    remeasured = {at.assignment_text(a): time_of(a)
                  for a in at.ParamSpace.make(axes).enumerate()}
    tuned = remeasured[at.assignment_text(result.best_assignment)]
    assert tuned <= 1.25 * min(remeasured.values())
    assert tuned < max(remeasured.values())


@pytest.mark.gpu
def test_tune_reduction_store_hit(pool, tmp_path, shared_cache):
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
    store = at.TuneStore(tmp_path)
    axes = {"unroll": (2, 8), "block": (256, 512)}
    cold = at.tune_reduction(spec, "dot_t", 1 << 22, axes, store=store, cache=shared_cache,
                             pool=pool)
    warm = at.tune_reduction(spec, "dot_t", 1 << 22, axes, store=store, cache=shared_cache,
                             pool=pool)
    assert warm.from_store and warm.best_assignment == cold.best_assignment
    assert all(e.status in ("ok", "pruned") for e in cold.table)


def test_size_buckets():
    assert at.size_bucket(1) == 1024 and at.size_bucket(1025) == 2048
    assert at.size_bucket(1 << 28) == 1 << 28 and at.size_bucket((1 << 28) + 1) == 1 << 29


@pytest.mark.gpu
def test_auto_kernels_tune_once_per_bucket(pool, tmp_path, shared_cache):
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    store = at.TuneStore(tmp_path)
    axes = {"unroll": (1, 4), "block": (128, 256)}
    k = at.AutoElementwise("float *x, float *z", "z[i] += x[i]", "acc_add", axes, store=store,
                           cache=shared_cache, pool=pool)
    x = nd.from_host(pool, nd.float32, np.ones(8000, np.float32))
    z = nd.from_host(pool, nd.float32, np.full(8000, 2.0, np.float32))
    k(x, z, n=5000)                  # tuning happens on synthetic data, not on z
    assert np.all(z.get()[:5000] == 3.0) and np.all(z.get()[5000:] == 2.0)
    k(x, z, n=8000)                  # same bucket (8192): no new campaign
    assert len(k.results) == 1 and k.results[8192].best_assignment in \
        at.ParamSpace.make(axes).enumerate()
    spec = rd.ReductionSpec("float *x", nd.float32, "0", "a + b")
    r = at.AutoReduction(spec, "auto_sum", axes, store=store, cache=shared_cache, pool=pool)
    assert float(r(x)) == 8000.0 and len(r.results) == 1
    again = at.AutoReduction(spec, "auto_sum", axes, store=store, cache=shared_cache, pool=pool)
    assert float(again(x)) == 8000.0 and again.results[8192].from_store


def test_algorithmic_bytes_follow_the_access_analysis():
    import ctypes
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    pool = nd.MemoryPool(lambda n: ctypes.create_string_buffer(n), zero_fill=lambda a, n: None)
    x, y, z = (pool.alloc(nd.float32, (1000,)) for _ in range(3))
    axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                                "z[i] = a * x[i] + b * y[i]", "axpy_bytes")
    assert at.algorithmic_bytes(axpy, 2.0, x, 3.0, y, z) == 12_000
    inplace = ew.ElementwiseKernel("float *x, float *z", "z[i] += x[i]", "inplace_bytes")
    assert at.algorithmic_bytes(inplace, x, z) == 12_000          # z read and written
    assert at.algorithmic_bytes(inplace, x, z, n=10) == 120
    dot = rd.dot_kernel(nd.float32)
    assert at.algorithmic_bytes(dot, x, y) == 8_000
    peak, kind = at.measured_hbm_gbs()
    assert peak > 1000 and kind in ("measured", "fallback")


def test_default_axes_add_prefetch_for_calls():
    assert "prefetch" not in at.default_axes("z[i] = a * x[i] + b * y[i]")
    assert "prefetch" not in at.default_axes("z[i] = (float) x[i] * 2")
    assert at.default_axes("z[i] = sin(x[i]) + 1")["prefetch"] == (False, True)
    assert at.default_axes("fabsf(x[i])")["prefetch"] == (False, True)
    assert at._check_axes(None, "exp(x[i])")["prefetch"] == (False, True)
    assert "prefetch" not in at._check_axes({"unroll": (1,)}, "exp(x[i])")
