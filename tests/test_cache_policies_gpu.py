"""Every load/store cache policy (``VariantParams.cache``) is a pure
performance knob: results are bit-identical to the default policy."""

import numpy as np
import pytest

from paper_0911_3456_b200 import _codegen as cg, elementwise as ew, ndarray as nd
from paper_0911_3456_b200 import reduction as rd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cache", sorted(cg.CACHE_POLICIES))
def test_policy_does_not_change_results(kernel_env, cache):
    kwargs, pool = kernel_env
    rng = np.random.default_rng(17)
    n = 1_000_003
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    hy = rng.uniform(-1, 1, n).astype(np.float32)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    outs = {}
    for c in ("default", cache):
        v = ew.VariantParams(cache=c, unroll=2)
        z = pool.alloc(nd.float32, (n,))
        ew.make_elementwise("float a, float *x, float b, float *y, float *z",
                            "z[i] = a * x[i] + b * y[i]", "axpy_pol", v, **kwargs)(
            2.0, x, -3.0, y, z)
        outs[c] = (z.get(), float(rd.dot_kernel(nd.float32, v, **kwargs)(x, y)))
    assert np.array_equal(outs["default"][0], outs[cache][0])
    if cache != "tma":       # the TMA fold walks tiles, not the strided order
        assert outs["default"][1] == outs[cache][1]
