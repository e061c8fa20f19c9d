"""The prelude's double sin / cos (templates/prelude.cuh ``rtcg_trig``),
emulated on the CPU with exact IEEE arithmetic from the constants the
prelude ships: every operation is a double multiply / add (Python floats,
round-to-nearest) or a fused multiply-add (exact rational, rounded once).
Pins the shipped coefficients and the shift-rounded quadrant without a GPU:
within 1 ulp of glibc (math.sin / math.cos) over several magnitudes and next
to multiples of pi/2.  The GPU test
``test_elementwise_gpu.py::test_double_sin_cos_bit_identical_to_cuda_library``
checks the kernel bits against CUDA's own sin / cos."""

import math
import re
import struct
from fractions import Fraction

import numpy as np
import pytest

from paper_0911_3456_b200 import _codegen as cg


def _constants():
    src = cg.template("prelude.cuh")

    def table(name):
        body = re.search(name + r"\[\d+\][^=]*=\s*\{(.*?)\};", src, re.S).group(1)
        return [float.fromhex(t.strip()) for t in body.split(",") if t.strip()]
    return table("rtcg_trig_k"), table("rtcg_trig_tab")


K, TAB = _constants()


def _fma(a: float, b: float, c: float) -> float:
    """fma rounded once; IEEE signed zeros (an exact zero sum is +0 unless
    both the product and the addend are -0)."""
    exact = Fraction(a) * Fraction(b) + Fraction(c)
    if exact == 0:
        prod_neg = (a == 0 or b == 0) and (math.copysign(1, a) * math.copysign(1, b) < 0)
        return -0.0 if prod_neg and math.copysign(1, c) < 0 else 0.0
    return float(exact)


# pi to 100 digits (the reduction constants must represent pi/2 far beyond a double)
PI = Fraction("3.1415926535897932384626433832795028841971693993751058209749445923078164062862089986280348253421170679")


def _lo32(d: float) -> int:
    v = struct.unpack("<q", struct.pack("<d", d))[0] & 0xFFFFFFFF
    return v - (1 << 32) if v & 0x80000000 else v


def _flip(v: float, q: int) -> float:
    if q & 2:
        bits = struct.unpack("<Q", struct.pack("<d", v))[0] ^ (1 << 63)
        return struct.unpack("<d", struct.pack("<Q", bits))[0]
    return v


def rtcg_trig(x: float, quadrant_shift: int) -> float:
    """Line for line the device function (fast path, |x| < 2^31)."""
    t = (x * K[0]) + K[1]
    q = _lo32(t) + quadrant_shift
    n = t - K[1]
    r = _fma(n, K[2], x)
    r = _fma(n, K[3], r)
    r = _fma(n, K[4], r)
    r2 = r * r
    row = TAB[8:16] if q & 1 else TAB[0:8]
    p = _fma(row[0], r2, row[1])
    for c in row[2:7]:
        p = _fma(p, r2, c)
    v = _fma(p, r2, K[5]) if q & 1 else _fma(p, r, r)
    return _flip(v, q)


def test_constants_shape():
    assert len(K) == 6 and len(TAB) == 16
    assert K[0] == float.fromhex("0x1.45f306dc9c883p-1")           # 2/pi rounded
    assert K[1] == 1.5 * 2.0**52
    # -(pi/2) in three parts: the parts sum to pi/2 well beyond double precision
    half_pi = Fraction(-K[2]) + Fraction(-K[3]) + Fraction(-K[4])
    assert abs(float(half_pi - PI / 2)) < 2.0**-150
    assert TAB[6] == 0.0 and TAB[14] == -0.5 and K[5] == 1.0


@pytest.mark.parametrize("fn, shift, ref", [("sin", 0, math.sin), ("cos", 1, math.cos)])
def test_emulated_prelude_trig_within_one_ulp_of_glibc(fn, shift, ref):
    rng = np.random.default_rng(7)
    k = np.arange(1, 400, dtype=np.float64)
    xs = np.concatenate([rng.uniform(-2, 2, 3000), rng.uniform(-1e4, 1e4, 1500),
                         rng.uniform(-2.0**31, 2.0**31, 500), k * (math.pi / 2),
                         np.nextafter(k * (math.pi / 2), 0), -k * math.pi,
                         [0.0, 1e-300, -5e-324, 2.0**-30]])
    worst = 0.0
    for x in xs.tolist():
        got, want = rtcg_trig(x, shift), ref(x)
        if got != want:
            worst = max(worst, abs(got - want) / math.ulp(abs(want)) if want else math.inf)
    assert worst <= 1.0, (fn, worst)


def test_emulated_sin_keeps_signed_zero():
    assert math.copysign(1.0, rtcg_trig(-0.0, 0)) == -1.0
    assert rtcg_trig(0.0, 0) == 0.0 and rtcg_trig(0.0, 1) == 1.0
