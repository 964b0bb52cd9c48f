import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


class CurandHost:
    """cuRAND's Philox4x32-10 compiled for the host (tests/pins); a library
    routine independent of the oracle, used to pin the oracle's generator and
    to build independent re-formulations in tests."""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        f = self.lib.curand_host_philox
        u32p = C.POINTER(C.c_uint32)
        f.argtypes = [u32p, u32p, u32p, C.c_long]
        f.restype = None

    def blocks(self, ctr, key):
        ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
        key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
        if key.shape[0] == 1 and ctr.shape[0] > 1:
            key = np.ascontiguousarray(np.repeat(key, ctr.shape[0], axis=0))
        out = np.zeros_like(ctr)
        u32p = C.POINTER(C.c_uint32)
        self.lib.curand_host_philox(ctr.ctypes.data_as(u32p), key.ctypes.data_as(u32p),
                                    out.ctypes.data_as(u32p), ctr.shape[0])
        return out

    # independent lane composition (R3/R4), vectorised with numpy
    def stream_blocks(self, seed, tag, b, t):
        b = np.asarray(b, dtype=np.uint64)
        ctr = np.stack([(b & 0xFFFFFFFF).astype(np.uint32), (b >> np.uint64(32)).astype(np.uint32),
                        np.full(b.shape, t, np.uint32), np.full(b.shape, tag, np.uint32)], axis=1)
        key = np.array([[seed & 0xFFFFFFFF, seed >> 32]], dtype=np.uint32)
        return self.blocks(ctr, key)

    def lane64(self, seed, tag, u, t):
        u = np.asarray(u, dtype=np.uint64)
        w = self.stream_blocks(seed, tag, u // np.uint64(2), t).astype(np.uint64)
        j = (u % np.uint64(2)).astype(np.int64) * 2
        rows = np.arange(u.size)
        return w[rows, j] | (w[rows, j + 1] << np.uint64(32))

    def lane32(self, seed, tag, u, t):
        u = np.asarray(u, dtype=np.uint64)
        w = self.stream_blocks(seed, tag, u // np.uint64(4), t)
        return w[np.arange(u.size), (u % np.uint64(4)).astype(np.int64)]


def mulhi64_bigint(x, n):
    """R6 with Python big integers (independent of the oracle's __int128)."""
    return np.array([(int(a) * int(n)) >> 64 for a in np.asarray(x).ravel()], dtype=np.int64)


@pytest.fixture(scope="session")
def curand_host(tmp_path_factory):
    d = tmp_path_factory.mktemp("pins")
    so = str(d / "libcurandhost.so")
    src = os.path.join(ROOT, "tests", "pins", "curand_philox_host.cpp")
    subprocess.check_call(["g++", "-O2", "-fPIC", "-shared", "-I/usr/local/cuda/include",
                           "-o", so, src])
    return CurandHost(so)
