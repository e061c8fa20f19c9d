"""Build ``oracle/_ref/`` from the reference itself -- TEST INFRASTRUCTURE ONLY.

Run in the build container, where /root/reference exists:

    python oracle/build_ref.py

For each benchmark kernel it calls the reference's OWN generator
(``rtcg.elementwise.generate`` / ``rtcg.reduction.generate_reduction_source``,
``src/elementwise.py:248-270``, ``src/reduction.py:133-181``) with the
reference's default variant (unroll=4, contiguous-blocks), and compiles the
emitted C with the reference's own command line (``cc -O2 -ffp-contract=off
-shared -fPIC``, ``src/jit.py:43,452-453``).  Outputs go to ``oracle/_ref/``
(git-ignored, shipped to the GPU box with the snapshot) with a manifest that
``oracle/refdrive.py`` uses to drive them exactly like the reference driver.
No reference source file is copied.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg/src")

# name -> (kind, signature, operation | (out, neutral, reduce, map))
KERNELS = {
    "axpy": ("elementwise", "float a, float *x, float b, float *y, float *z",
             "z[i] = a * x[i] + b * y[i]"),
    "polysin": ("elementwise", "double a, double *x, double *z",
                "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"),
    "dot_k": ("reduction", "float *x, float *y", ("float32", "0", "a + b", "x[i] * y[i]")),
    "maxabs": ("reduction", "float *x", ("float32", "0", "a > b ? a : b", "fabsf(x[i])")),
    "sumsq": ("reduction", "float *x", ("float32", "0", "a + b", "x[i] * x[i]")),
    "sum_i64": ("reduction", "int64_t *x", ("int64", "0", "a + b", None)),
}


def main() -> int:
    if not REF_SRC.is_dir():
        print("reference tree absent; oracle/_ref not rebuilt", file=sys.stderr)
        return 1
    os.environ.setdefault("RTCG_CACHE_DIR", tempfile.mkdtemp(prefix="rtcg-ref-"))
    sys.path.insert(0, str(REF_SRC))
    from rtcg import elementwise as ew, ndarray as nd, reduction as rd  # noqa: E402
    from rtcg import jit  # noqa: E402

    OUT.mkdir(exist_ok=True)
    cc = jit.ToolchainConfig()  # reference defaults: cc -O2 -ffp-contract=off
    variant = ew.VariantParams(unroll=4, workers=1)
    manifest = {"compiler": [cc.cc, *cc.flags, "-shared", "-fPIC"],
                "toolchain": cc.resolved_identity(), "variant": {"unroll": 4,
                                                                 "chunking": "contiguous-blocks"},
                "kernels": {}}
    for name, (kind, sig, what) in KERNELS.items():
        if kind == "elementwise":
            source = ew.generate(ew.parse_signature(sig), what, name, variant)
            entry = {"kind": kind, "signature": sig, "operation": what}
        else:
            out, neutral, reduce_expr, map_expr = what
            spec = rd.ReductionSpec(sig, nd.BY_NAME[out], neutral, reduce_expr, map_expr)
            source = rd.generate_reduction_source(spec, name, variant)
            entry = {"kind": kind, "signature": sig, "out": out,
                     "acc": spec.acc_dtype.name, "neutral": neutral}
        c_path = OUT / f"{name}.c"
        so_path = OUT / f"{name}.so"
        c_path.write_text(source)
        subprocess.run([cc.cc, *cc.flags, "-shared", "-fPIC", "-o", str(so_path), str(c_path),
                        "-lm"], check=True)
        manifest["kernels"][name] = entry
        print(so_path)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
