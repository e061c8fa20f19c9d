import sys, time, statistics
sys.path.insert(0, '/root/repo')
from paper_0911_3456_b200 import elementwise as ew, _runtime as rt, jit
sig = ew.parse_signature("double *x, double *z")
def strip_general(src):
    i = src.index('// General path')
    j = src.index('// Vector path')
    return src[:i] + src[j:]
for label, tf in (("both", lambda s: s), ("vector_only", strip_general), ("both2", lambda s: s)):
    ts = []
    for k in range(8):
        src = tf(ew.generate(sig, f"z[i] = {k + 1000 * len(label)} * x[i] + {k + 1}", f"affine_{k}", ew.VariantParams()))
        t0 = time.perf_counter(); rt.compile_cubin(src, jit.DEFAULT_FLAGS); ts.append(time.perf_counter() - t0)
    print(label, round(statistics.median(ts) * 1e3, 1), [round(t * 1e3) for t in ts])
