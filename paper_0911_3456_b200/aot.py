"""Stock kernel instantiations of the templates (the benchmark set).

``stock_sources()`` renders them to CUDA C++; ``_build.build_prebuilt`` feeds
those to nvcc for sm_100a (SASS inspection without a GPU) and
``compile_stock()`` warms the NVRTC cubin cache with the same sources.
"""

from __future__ import annotations

from . import elementwise as ew
from . import jit
from . import ndarray as nd
from . import reduction as rd

ELEMENTWISE = {
    "axpy": ("float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]"),
    "polysin": ("double a, double *x, double *z",
                "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"),
}
REDUCTIONS = {
    "dot_k": ("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]"),
    "maxabs": ("float *x", nd.float32, "0", "a > b ? a : b", "fabsf(x[i])"),
    "sumsq": ("float *x", nd.float32, "0", "a + b", "x[i] * x[i]"),
    "sum_k": ("int64_t *x", nd.int64, "0", "a + b", None),
}


def stock_sources(variant: ew.VariantParams | None = None) -> dict:
    variant = variant or ew.VariantParams()
    out = {}
    for name, (sig, op) in ELEMENTWISE.items():
        # what ElementwiseKernel compiles: the vector entry eagerly, the
        # general entry on first need
        out[name] = ew.generate(ew.parse_signature(sig), op, name, variant, entries="vector")
        out[f"{name}_g"] = ew.generate(ew.parse_signature(sig), op, name, variant,
                                       entries="general")
    for name, (sig, dt, neutral, red, mp) in REDUCTIONS.items():
        spec = rd.ReductionSpec(sig, dt, neutral, red, mp)
        out[name] = rd.generate_reduction_source(spec, name, variant, entries="vector")
        out[f"{name}_g"] = rd.generate_reduction_source(spec, name, variant, entries="general")
    return out


def compile_stock(config: jit.ToolchainConfig | None = None, cache=None) -> dict:
    return {name: jit.compile(src, config, cache) for name, src in stock_sources().items()}
