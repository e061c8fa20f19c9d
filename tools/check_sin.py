"""Exact-arithmetic check (fractions) of a branch-free fdlibm-style double
sin (3-term FMA Cody-Waite reduction, both fdlibm polynomials, quadrant
select) against glibc math.sin: max 1 ulp over |x| < 2, 100, 2^19 and next to
multiples of pi/2.  Tried as a replacement for CUDA's sin in generated
kernels and rejected: evaluating both polynomials costs 33 FP64 instructions
per element against CUDA's 21 (table-selected coefficients), so the C3 kernel
got slower (5.0 vs 5.8 TB/s)."""
from fractions import Fraction as F
import math, random, struct
PI = F("3.14159265358979323846264338327950288419716939937510582097494459230781640628620899862803482534211706798214808651328230664709384460955058223172535940812848111745028410270193852110555964462294895493038196")
half = PI / 2
def rnd(f):  # nearest double to a Fraction
    return float(f) if True else None
P1 = float(half); P2 = float(half - F(P1)); P3 = float(half - F(P1) - F(P2))
print("P1", P1.hex(), "P2", P2.hex(), "P3", P3.hex())
TWO_OVER_PI = float(2 / PI)
print("2/pi", TWO_OVER_PI.hex())
def fma(a, b, c):
    return float(F(a) * F(b) + F(c))
S = [-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
     2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10]
C = [4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
     -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11]
MAGIC = 6755399441055744.0  # 0x1.8p52
def lo32(d):
    return struct.unpack("<q", struct.pack("<d", d))[0] & 0xffffffff
def mysin(x):
    t = fma(x, TWO_OVER_PI, MAGIC)
    q = lo32(t)
    n = t - MAGIC
    r = fma(-n, P1, x); r = fma(-n, P2, r); r = fma(-n, P3, r)
    z = r * r
    rs = fma(z, fma(z, fma(z, fma(z, S[5], S[4]), S[3]), S[2]), S[1])
    s = fma(z * r, fma(z, rs, S[0]), r)
    rc = z * fma(z, fma(z, fma(z, fma(z, fma(z, C[5], C[4]), C[3]), C[2]), C[1]), C[0])
    hz = 0.5 * z
    w = 1.0 - hz
    c = w + (((1.0 - w) - hz) + z * rc)
    v = c if q & 1 else s
    return -v if q & 2 else v
def ulp_err(got, want):
    if got == want: return 0.0
    return abs(got - want) / math.ulp(want)
random.seed(1)
worst = 0
for rng in (2.0, 100.0, 2.0**19):
    w = 0
    for _ in range(20000):
        x = random.uniform(-rng, rng)
        e = ulp_err(mysin(x), math.sin(x))
        w = max(w, e)
    print("range", rng, "max ulp vs glibc", w)
# near multiples of pi/2
w = 0
for k in range(1, 2000):
    x = float(k * half)
    for d in (x, math.nextafter(x, 0), math.nextafter(x, 10**9)):
        w = max(w, ulp_err(mysin(d), math.sin(d)))
print("near k*pi/2 max ulp", w)
