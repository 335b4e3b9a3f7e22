"""GPU parity of the sharded steady-state step (paper_2604_25899_b200/steady_shard.py) at
world 1, 2 and 4 (when the box has the GPUs) against the unmodified reference on the whole
cluster (tests/steady_shard_worker.py)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

from oracle.py_oracle import reference_available

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_steady_matches_reference(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    if not reference_available(16):
        pytest.skip("oracle/_ref not built")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), os.path.join(ROOT, "tests", "steady_shard_worker.py")]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-6000:]
    assert "steady shard parity ok" in p.stdout, p.stdout[-3000:]
