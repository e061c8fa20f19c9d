"""paper_0911_3456_b200 -- B200-native run-time code generation (RTCG) toolkit.

A from-scratch sm_100a implementation of the data-parallel hot path of
rtcg-kit (arXiv 0911.3456, PyCUDA/PyOpenCL): user C expressions become CUDA
kernels (``ElementwiseKernel``, ``ReductionKernel``) compiled by NVRTC into a
content-addressed cubin cache and launched on ``GPUArray`` device arrays, with
an autotuner over block size / unroll and NCCL-combined multi-GPU reductions.

Module layout mirrors the reference package ``rtcg``: ``ndarray``,
``elementwise``, ``reduction``, ``jit``, ``autotune``, ``csyntax``; plus
``parallel`` (multi-GPU sharding) and ``_runtime`` (the C-ABI binding).
"""

from ._version import TOOLKIT_VERSION

__version__ = TOOLKIT_VERSION
__all__ = ["TOOLKIT_VERSION"]
