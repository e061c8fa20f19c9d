import os
import sys
from pathlib import Path

import hypothesis
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

hypothesis.settings.register_profile("default", deadline=None, max_examples=60)
hypothesis.settings.load_profile("default")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_runtime():
    from paper_0911_3456_b200 import _build
    _build.build_runtime()
    _build.build_fastlaunch()


_ensure_runtime()


def have_gpu() -> bool:
    from paper_0911_3456_b200 import _runtime
    return _runtime.have_gpu()


def pytest_collection_modifyitems(config, items):
    if have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _sandbox_caches(tmp_path_factory):
    """Keep the cubin / tuning caches inside the test tmp tree."""
    root = tmp_path_factory.mktemp("default-cache")
    old = os.environ.get("RTCG_CACHE_DIR")
    os.environ["RTCG_CACHE_DIR"] = str(root)
    yield
    if old is None:
        os.environ.pop("RTCG_CACHE_DIR", None)
    else:
        os.environ["RTCG_CACHE_DIR"] = old


@pytest.fixture(scope="session")
def toolchain():
    from paper_0911_3456_b200 import jit
    return jit.ToolchainConfig()


@pytest.fixture()
def cache(tmp_path):
    from paper_0911_3456_b200 import jit
    return jit.CacheStore(tmp_path / "cache")


@pytest.fixture(scope="session")
def shared_cache(tmp_path_factory):
    from paper_0911_3456_b200 import jit
    return jit.CacheStore(tmp_path_factory.mktemp("shared-cache"))


@pytest.fixture()
def pool():
    """A fresh device pool (GPU tests only)."""
    from paper_0911_3456_b200 import _runtime, ndarray
    _runtime.set_device(0)
    p = ndarray.MemoryPool(device=0)
    yield p
    _runtime.synchronize()
    p.release_free()


@pytest.fixture()
def kernel_env(shared_cache, toolchain, pool):
    return {"cache": shared_cache, "config": toolchain}, pool


@pytest.fixture(scope="session")
def golden():
    import json
    return json.loads((ROOT / "tests" / "golden" / "reference_outputs.json").read_text())
