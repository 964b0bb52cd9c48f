"""Cross-process peer-memory exchange on one B200: two
or three processes, one GPU, gloo host collectives.  The sharded wealth step's P2P path
-- cudaIpcGetMemHandle / cudaIpcOpenMemHandle of the bucket blocks and
wealth_recv_p2p_kernel reading the OTHER process's buckets -- must equal the
unsharded oracle bit for bit (column, all-reduced total / active / digest),
including the collective overflow replay with 2-bit counters."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["dense", "sparse"])
@pytest.mark.parametrize("world,n,steps,bits", [(2, 200_003, 12, 4), (2, 90_001, 10, 2), (3, 150_001, 9, 4)])
def test_multi_process_ipc_exchange_bit_exact(tmp_path, monkeypatch, world, n, steps, bits, mode):
    # dense (default up to 8 ranks): the owners sum the other processes' global
    # counters; sparse: they read the other processes' id buckets
    monkeypatch.setenv("AMBER_WEALTH_EXCHANGE", mode)
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, "tests", "mp_wealth_ipc_worker.py"), str(out), str(n), "77", str(steps), str(bits)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=dict(os.environ))
    errs = [ln for ln in (r.stdout + r.stderr).splitlines() if "AmberError" in ln or "Error:" in ln]
    assert r.returncode == 0, "\n".join(errs[:10]) + "\n" + r.stderr[-2000:]
    res = json.load(open(out))
    assert res["exchange"] == {"dense": 3, "sparse": 2}[mode], res  # the P2P (IPC-mapped) exchange ran
    assert res["column_equal"] and res["total_equal"] and res["active_equal"] and res["digest_equal"], res
    if bits == 2:
        assert res["replays"] > 0, res  # overflow detected and replayed on both ranks together
