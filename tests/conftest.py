import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    # Build the native pieces if a fresh checkout has not been built yet
    # (the package refuses to import without libgaes_b200.so).
    if not os.path.exists(os.path.join(REPO, "paper_1506_08503_b200", "libgaes_b200.so")):
        import __graft_entry__
        __graft_entry__._load_build_module().build()
    from oracle import oracle as _oracle
    _oracle.build()


@pytest.fixture(scope="session")
def golden():
    with np.load(os.path.join(GOLDEN_DIR, "golden.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_meta():
    import json
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


def reference_package_dir():
    """baseline/_ref (pip-installed reference, ships to the GPU box) if present."""
    d = os.path.join(REPO, "baseline", "_ref")
    return d if os.path.isdir(os.path.join(d, "gaes")) else None
