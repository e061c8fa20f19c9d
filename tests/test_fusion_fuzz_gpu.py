"""Seeded random GPUArray operator chains: the fused kernel, the eager GPU
chain and the oracle's eager chain (``oracle/chain.py``: each operator one
reference kernel, C semantics) must store the same bits.

Chains mix 2-3 arrays of random dtypes with Python ints, Python floats and
numpy scalars on either side of + - * /.  Undefined behaviour is avoided by
construction: array values are 1..20 and scalars nonzero, divisors are
always leaves (never a difference that could be zero), depth <= 3 keeps
signed arithmetic far from overflow, and the promotion rules never convert a
negative or fractional value to an unsigned type."""

import numpy as np
import pytest

from oracle import chain as och
from paper_0911_3456_b200 import fusion, ndarray as nd

pytestmark = pytest.mark.gpu

_DT = ("int8", "int16", "int32", "int64", "uint8", "uint16", "uint32", "uint64", "float32",
       "float64")


def _tree(rng, leaves, depth):
    if depth == 0 or rng.random() < 0.3:
        if rng.random() < 0.25:
            kind = rng.integers(0, 3)
            if kind == 0:
                return ("s", int(rng.integers(1, 9)))
            if kind == 1:
                return ("s", float(rng.choice([0.5, 1.25, 3.0])))
            return ("s", np.dtype(rng.choice(["int16", "float32", "uint8"])).type(3))
        return ("a", int(rng.integers(0, leaves)))
    op = ("+", "-", "*", "/")[rng.integers(0, 4)]
    left, right = _tree(rng, leaves, depth - 1), _tree(rng, leaves, depth - 1)
    if op == "/" and right[0] not in ("a", "s"):
        right = ("a", int(rng.integers(0, leaves)))     # divisors: nonzero leaves only
    if left[0] == "s" and right[0] == "s":
        right = ("a", 0)
    return (op, left, right)


def _apply(node, arrays):
    if node[0] == "a":
        return arrays[node[1]]
    if node[0] == "s":
        return node[1]
    a, b = _apply(node[1], arrays), _apply(node[2], arrays)
    return {"+": lambda: a + b, "-": lambda: a - b, "*": lambda: a * b,
            "/": lambda: a / b}[node[0]]()


@pytest.mark.parametrize("seed", range(40))
def test_random_chains_fused_eager_oracle(pool, seed):
    rng = np.random.default_rng(1000 + seed)
    count = int(rng.integers(2, 4))
    names = [str(rng.choice(_DT)) for _ in range(count)]
    n = int(rng.choice([1, 7, 4099, 100_003]))
    host = [rng.integers(1, 21, n).astype(name) for name in names]
    dev = [nd.from_host(pool, nd.BY_NAME[name], h) for name, h in zip(names, host)]
    tree = _tree(rng, count, int(rng.integers(1, 4)))
    if tree[0] in ("a", "s"):
        tree = ("+", tree, ("a", count - 1))
    try:
        want = _apply(tree, [och.HostArray(h) for h in host])
    except ZeroDivisionError:
        pytest.skip("integer division by a scalar zero (raised on both sides)")
    if not isinstance(want, och.HostArray):
        pytest.skip("scalar-only tree")
    want = want.values
    eager = _apply(tree, dev)
    lazy = _apply(tree, [fusion.lazy(d) for d in dev])
    fused = fusion.evaluate(lazy)
    assert fused.dtype.name == eager.dtype.name == want.dtype.name
    got_f, got_e = fused.get(), eager.get()
    assert got_f.tobytes() == want.tobytes(), (names, tree)
    assert got_e.tobytes() == want.tobytes(), (names, tree)
