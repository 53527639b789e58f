import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line(
        "markers", "slow: seconds-long CPU oracle run at config size")


def _ensure_built() -> None:
    """Build libgf2b200.so and the oracle's C port if a fresh checkout lacks
    them (the built files are git-ignored); nvcc cross-compiles without a GPU."""
    import subprocess
    lib = os.path.join(ROOT, "paper_0811_1714_b200", "libgf2b200.so")
    port = os.path.join(ROOT, "oracle", "libgf2oracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j4", "-C", os.path.join(ROOT, "paper_0811_1714_b200", "csrc")],
                       check=True)
    if not os.path.exists(port):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def digests():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "digests.json")) as fh:
        return json.load(fh)
