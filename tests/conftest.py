import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (run on the B200 box)")
    _ensure_library()


def _ensure_library():
    """Build libadct_cuda.so in-tree if it is missing (fresh checkout: the .so
    is git-ignored).  Needs nvcc; without it the C-ABI tests fail loudly."""
    lib = os.path.join(ROOT, "paper_1702_00817_b200", "libadct_cuda.so")
    if os.environ.get("ADCT_LIB_PATH") or os.path.exists(lib):
        return
    import shutil
    import subprocess

    if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
        return
    env = dict(os.environ)
    env["PATH"] = env.get("PATH", "") + ":/usr/local/cuda/bin"
    subprocess.run(["make", "-j8"], cwd=os.path.join(ROOT, "paper_1702_00817_b200", "csrc"), env=env,
                   check=True, stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def reference():
    """The live reference package `adct` (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference sources not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import adct

    return adct


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
