"""CUDA-graph capture of generated-kernel sequences.

Small problems (C5's n = 2^16..2^22) are bound by per-launch host cost
(~10 us per call through Python), not by HBM.  Capturing a chain once and
replaying it as one graph launch removes that cost:

    g = graph.Graph()
    with g.capture():
        axpy(2.0, x, -3.0, y, z)          # any ElementwiseKernel / fused / reduction launch
        dot.launch(z, z, out=result)      # reductions: device-side result only
    for _ in range(1000):
        g.launch()                        # one cuGraphLaunch per replay
    g.synchronize()

Arguments are frozen at capture time (the same arrays and scalars are used on
every replay), exactly like any CUDA graph.  Host synchronisation (``get()``,
numpy-returning reductions) is not allowed inside a capture; allocations made
inside it (operator outputs) stay owned by the graph's arrays.
"""

from __future__ import annotations

from contextlib import contextmanager

from . import _runtime

__all__ = ["Graph"]


class Graph:
    """A captured, instantiated launch sequence replayable on its stream."""

    def __init__(self, stream: _runtime.Stream | None = None) -> None:
        self.stream = stream or _runtime.Stream()
        if not self.stream.handle:
            raise ValueError("graphs need a created stream, not the legacy default stream")
        self.handle = 0
        self.keepalive: list = []

    @contextmanager
    def capture(self):
        """Route this thread's launches to the graph's stream and record them."""
        if self.handle:
            raise RuntimeError("graph already captured")
        _runtime.begin_capture(self.stream.handle)
        ok = False
        try:
            with _runtime.use_stream(self.stream.handle):
                yield self
            ok = True
        finally:
            graph = _runtime.end_capture(self.stream.handle)
            if ok:
                self.handle = graph
            elif graph:
                _runtime.graph_destroy(graph)

    def keep(self, *objects) -> None:
        """Hold references (arrays created inside the capture) for the graph's
        lifetime."""
        self.keepalive.extend(objects)

    def launch(self) -> None:
        if not self.handle:
            raise RuntimeError("graph has not been captured")
        _runtime.graph_launch(self.handle, self.stream.handle)

    def synchronize(self) -> None:
        self.stream.synchronize()

    def close(self) -> None:
        if self.handle:
            _runtime.graph_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
