"""The README's usage examples run as written (smaller sizes)."""

import re
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_readme_python_blocks_run():
    text = (Path(__file__).resolve().parent.parent / "README.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    assert len(blocks) >= 2
    code = "\n".join(blocks).replace("1 << 28", "1 << 20").replace("1 << 26", "1 << 18")
    scope: dict = {}
    exec(compile(code, "README.md", "exec"), scope)      # noqa: S102 - our own docs
    x, y, w, out, h = (scope[k] for k in ("x", "y", "w", "out", "h"))
    assert np.array_equal(w.get(), (x.get() * 2 + y.get()) - x.get())
    assert np.allclose(out, np.sin(h), rtol=0, atol=4 * np.spacing(1.0))
    assert float(scope["s"].get()) == pytest.approx(
        float(np.sum(x.get().astype(np.float64) * y.get() + 1.0)), rel=1e-9)
