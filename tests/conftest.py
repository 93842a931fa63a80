import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libgns.so)")
    config.addinivalue_line("markers", "slow: long-running statistical test")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "gnsbench"))


@pytest.fixture(scope="session")
def gb():
    """The reference package (only in the build container)."""
    if not reference_available():
        pytest.skip("reference package not present (GPU box); golden fixtures cover it")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import gnsbench
    return gnsbench


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    out = {}
    for name in ("kat", "sampler", "model"):
        with np.load(os.path.join(GOLDEN, f"golden_{name}.npz")) as z:
            out[name] = {k: z[k] for k in z.files}
    return out
