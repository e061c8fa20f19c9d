"""PyCUDA ``driver`` argument handlers for host data: ``In``, ``Out``,
``InOut``.

Passing a host numpy array wrapped in one of these to an
:class:`~paper_0911_3456_b200.elementwise.ElementwiseKernel` turns the call
into a streamed host call: the index space is cut into chunks, and chunk j's
host-to-device copies, kernel and device-to-host copies run on one of two
CUDA streams, so with page-locked host buffers the upload of chunk j+1, the
kernel of chunk j and the download of chunk j-1 overlap (PCIe is full duplex
and the B200 has separate copy engines per direction).  The call returns when
every ``Out`` / ``InOut`` array holds its result.  ``GPUArray`` arguments may
be mixed in; they are indexed globally as usual.
"""

from __future__ import annotations

import numpy as np

__all__ = ["In", "Out", "InOut", "HostArg"]


class HostArg:
    """A host array argument with a transfer direction."""

    copy_in = False
    copy_out = False

    def __init__(self, array) -> None:
        if not isinstance(array, np.ndarray):
            raise TypeError(f"{type(self).__name__} wraps a numpy array")
        if not array.flags.c_contiguous:
            raise ValueError(f"{type(self).__name__} needs a C-contiguous array")
        if self.copy_out and not array.flags.writeable:
            raise ValueError(f"{type(self).__name__} needs a writeable array")
        self.array = array

    @property
    def size(self) -> int:
        return self.array.size

    def __repr__(self) -> str:
        return f"{type(self).__name__}({self.array.dtype}[{self.array.size}])"


class In(HostArg):
    """Host input: copied to the device before the kernel reads it."""
    copy_in = True


class Out(HostArg):
    """Host output: filled from the device after the kernel writes it."""
    copy_out = True


class InOut(HostArg):
    """Host array read and written by the kernel."""
    copy_in = True
    copy_out = True
