"""Replacement for the closed compute-sanitizer: the
bounds build (libamber_bounds.so, -DAMBER_BOUNDS: device-side checks on every
computed counter word, CSR arc, neighbour id, cell run and sorted slot) run
with AMBER_SYNC_DEBUG=1 (a device synchronize + error check after every
launch) over a small run of every kernel family (tools/sanitize_small.py) and
the sharded loopback tests.  A failed check traps the kernel and the run
fails, naming the launch."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2601_16292_b200", "libamber_bounds.so")

pytestmark = pytest.mark.gpu


def env():
    if not os.path.exists(LIB):
        from paper_2601_16292_b200 import build
        build.build(bounds=True)
    e = dict(os.environ, AMBER_LIB_PATH=LIB, AMBER_SYNC_DEBUG="1")
    return e


def test_every_kernel_family_under_bounds_checks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_small.py")], env=env(),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "sanitize run ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "AMBER_BOUNDS" not in r.stdout + r.stderr


def test_sharded_and_sir_parity_under_bounds_checks():
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_sharded.py"),
                        os.path.join(ROOT, "tests", "test_gpu_sir.py") + "::test_forced_direction_every_step_ragged"],
                       env=env(), capture_output=True, text=True, timeout=1500, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "AMBER_BOUNDS" not in r.stdout + r.stderr
