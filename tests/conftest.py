import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"

# Parity tests compare runs bit for bit (layouts, env switches, subprocesses):
# compile generated stencils on first use so every call of a layer runs the
# same kernel.  The default background mode has its own test
# (test_gpu_engine.py::test_jit_async_first_call).
os.environ.setdefault("SKC_JIT", "sync")
# share compiled stencils with the subprocess tests (the on-disk cache is
# opt-in; a private 0700 directory per session)
if "SKC_CACHE_DIR" not in os.environ:
    import tempfile
    os.environ["SKC_CACHE_DIR"] = tempfile.mkdtemp(prefix="skc_cache_")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


def split_layers(off, w, layout):
    layers, base = [], 0
    for n in np.asarray(layout).tolist():
        layers.append((off[base:base + n], w[base:base + n]))
        base += n
    return layers


def normwise(a, b):
    """max|a-b| / max|b| (SURVEY D7 tolerance definition)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(float(np.abs(b).max(initial=0.0)), 1e-300)
    return float(np.abs(a - b).max(initial=0.0)) / den
