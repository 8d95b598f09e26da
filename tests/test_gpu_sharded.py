"""The KV-head sharded certified step on one GPU (2 ranks, gloo; the driver's
runs have one B200): gathered outputs and certificates equal the unsharded
step bit for bit, and a canary trip on rank 1 makes its layer dense on rank 0
(tests/sharded_worker.py)."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_equals_unsharded(world):
    import __graft_entry__
    __graft_entry__.build()  # once, before the ranks start
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), os.path.join(HERE, "sharded_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"SHARDED OK world={world}" in r.stdout
