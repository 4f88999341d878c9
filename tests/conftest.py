import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def curand_philox_ref(tmp_path_factory):
    """Host build of cuRAND's curand_Philox4x32_10 (tests/tools)."""
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the cuRAND host reference")
    out = tmp_path_factory.mktemp("philox") / "philox_ref"
    src = os.path.join(ROOT, "tests", "tools", "curand_philox_ref.cu")
    subprocess.run([nvcc, "-Wno-deprecated-gpu-targets", "-o", str(out), src],
                   check=True, capture_output=True)
    return str(out)
