"""numpy restatement of per-element C semantics -- TEST INFRASTRUCTURE ONLY.

Mirrors the acceptance corpus of the reference (``tests/test_acceptance.py``:
ops ``:100-112``, sizes/variants ``:114-116``, C-semantics oracle ``:119-163``,
operand recipe ``:166-179``) and states the float-reduction tolerance used
for this path.
"""

from __future__ import annotations

import math

import numpy as np

# (name, operand shape, statement); "axy" has a leading scalar a (= 3)
CORPUS_OPS = (
    ("add", "xy", "z[i] = x[i] + y[i]"),
    ("sub", "xy", "z[i] = x[i] - y[i]"),
    ("mul", "xy", "z[i] = x[i] * y[i]"),
    ("div", "xy", "z[i] = x[i] / y[i]"),
    ("min2", "xy", "z[i] = x[i] < y[i] ? x[i] : y[i]"),
    ("max2", "xy", "z[i] = x[i] > y[i] ? x[i] : y[i]"),
    ("diff2", "xy", "z[i] = (x[i] - y[i]) * (x[i] + y[i])"),
    ("saxpy", "axy", "z[i] = a * x[i] + y[i]"),
    ("scale", "x", "z[i] = 3 * x[i]"),
    ("incr", "x", "z[i] = x[i] + 1"),
    ("half", "x", "z[i] = x[i] / 2"),
)
CORPUS_SIZES = (0, 1, 7, 1000, 10**6)
CORPUS_SEED = 2024
DTYPE_NAMES = ("int8", "int16", "int32", "int64", "uint8", "uint16", "uint32", "uint64",
               "float32", "float64")
CNAMES = {"int8": "int8_t", "int16": "int16_t", "int32": "int32_t", "int64": "int64_t",
          "uint8": "uint8_t", "uint16": "uint16_t", "uint32": "uint32_t",
          "uint64": "uint64_t", "float32": "float", "float64": "double"}


def corpus_signature(shape: str, cname: str) -> str:
    return {"xy": f"{cname} *x, {cname} *y, {cname} *z",
            "axy": f"{cname} a, {cname} *x, {cname} *y, {cname} *z",
            "x": f"{cname} *x, {cname} *z"}[shape]


def corpus_operands(dtype_names=DTYPE_NAMES, seed: int = CORPUS_SEED):
    """{dtype: (x, y)} of length max(CORPUS_SIZES); one generator walked in
    dtype order, so every dtype's draw matches the reference test's."""
    rng = np.random.default_rng(seed)
    n = max(CORPUS_SIZES)
    out = {}
    for name in dtype_names:
        dt = np.dtype(name)
        if dt.kind == "f":
            x = rng.uniform(-2.0, 2.0, size=n).astype(dt)
            y = rng.uniform(0.5, 2.0, size=n).astype(dt)
        elif dt.kind == "i":
            x = rng.integers(-100, 101, size=n).astype(dt)
            sign = rng.integers(0, 2, size=n) * 2 - 1
            y = (rng.integers(1, 101, size=n) * sign).astype(dt)
        else:
            x = rng.integers(0, 201, size=n).astype(dt)
            y = rng.integers(1, 101, size=n).astype(dt)
        out[name] = (x, y)
    return out


def c_elementwise(op: str, x, y, dtype_name: str):
    """What the generated C computes per element, in numpy."""
    dt = np.dtype(dtype_name)
    if dt.kind == "f":
        t = dt.type
        table = {
            "add": lambda: x + y, "sub": lambda: x - y, "mul": lambda: x * y,
            "div": lambda: x / y, "min2": lambda: np.where(x < y, x, y),
            "max2": lambda: np.where(x > y, x, y), "diff2": lambda: (x - y) * (x + y),
            "saxpy": lambda: t(3) * x + y, "scale": lambda: t(3) * x,
            "incr": lambda: x + t(1), "half": lambda: x / t(2),
        }
        return table[op]()
    # integers: C promotes to int (or wider) then narrows on store; computing
    # in 64 bits and truncating gives the same bits for this corpus
    wide = np.int64 if dt.kind == "i" else np.uint64
    wx, wy = x.astype(wide), y.astype(wide)

    def cdiv(a, b):
        if dt.kind == "u":
            return a // b
        q = np.abs(a) // np.abs(b)
        return np.where((a < 0) ^ (np.asarray(b) < 0), -q, q)

    table = {
        "add": lambda: wx + wy, "sub": lambda: wx - wy, "mul": lambda: wx * wy,
        "div": lambda: cdiv(wx, wy), "min2": lambda: np.where(wx < wy, wx, wy),
        "max2": lambda: np.where(wx > wy, wx, wy), "diff2": lambda: (wx - wy) * (wx + wy),
        "saxpy": lambda: wide(3) * wx + wy, "scale": lambda: wide(3) * wx,
        "incr": lambda: wx + wide(1), "half": lambda: cdiv(wx, wide(2)),
    }
    with np.errstate(over="ignore"):
        return table[op]().astype(dt)


def float_reduction_bound(terms, result_dtype: str) -> float:
    """|got - fsum(terms)| allowed for an fp64-accumulated reduction whose
    result is rounded to *result_dtype*:  1/2 ulp of the result plus
    n * 2**-53 * sum|terms|  (order-of-accumulation error)."""
    terms = np.asarray(terms, dtype=np.float64)
    exact = math.fsum(terms.tolist()) if terms.size < 5_000_000 else float(np.sum(terms))
    half_ulp = 0.5 * float(np.spacing(np.abs(np.dtype(result_dtype).type(exact))))
    return half_ulp + terms.size * 2.0 ** -53 * float(np.sum(np.abs(terms)))


def exact_sum(terms) -> float:
    return math.fsum(np.asarray(terms, dtype=np.float64).tolist())


# --- exact sums of float32 values at any n (what math.fsum gives, in seconds) ---------------
#
# A float32 value is m * 2^(e-24) with an integer |m| < 2^24 (frexp).  Summing
# the integer mantissas per exponent is exact in float64 while a bucket's sum
# stays below 2^53 (chunks of <= 2^28 values); buckets are carried in int64
# across chunks and combined in Python integers.

_EOFF, _EBINS = 160, 320


def f32_buckets(values, chunk: int = 1 << 24) -> np.ndarray:
    """Per-exponent integer mantissa sums of float32 values (exact)."""
    values = np.asarray(values, dtype=np.float32).reshape(-1)
    total = np.zeros(_EBINS, np.int64)
    for lo in range(0, values.size, chunk):
        m, e = np.frexp(values[lo:lo + chunk])
        mi = np.ldexp(m.astype(np.float64), 24)
        total += np.bincount(e.astype(np.int64) + _EOFF, weights=mi,
                             minlength=_EBINS).astype(np.int64)
    return total


def buckets_fraction(buckets):
    from fractions import Fraction
    num = 0
    for k, s in enumerate(np.asarray(buckets, dtype=np.int64).tolist()):
        if s:
            num += int(s) << k
    return Fraction(num, 1 << (_EOFF + 24))


def exact_f32_sum(values) -> float:
    """Correctly rounded float64 of the exact sum of float32 values --
    ``math.fsum(values)`` without a Python loop."""
    return float(buckets_fraction(f32_buckets(values)))
