"""T1 RNG cross-check: the product's device Philox against cuRAND's
device routine on 2^20 random (counter, key) pairs, plus the receiver
arithmetic (tests/pins/philox_device_check.cu, compiled here with nvcc)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_device_philox_equals_curand(tmp_path):
    exe = str(tmp_path / "philox_check")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                           "-I", os.path.join(ROOT, "paper_2601_16292_b200", "csrc"), "-o", exe,
                           os.path.join(ROOT, "tests", "pins", "philox_device_check.cu")])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "philox_mismatch 0 mulhi_mismatch 0 lane_mismatch 0" in r.stdout
