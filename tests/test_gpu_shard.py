"""GPU parity of the multi-GPU sharded step (paper_2604_25899_b200/shard.py): every rank's
share of decisions, admissions, tiers and the replicated L3 must equal the single-cluster
oracle.  World 1 always runs (the NCCL plumbing with one rank); world 2/4 run when the box
has that many GPUs (gpurun --gpus N)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_step_matches_oracle(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), os.path.join(ROOT, "tests", "shard_worker.py")]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-6000:]
    assert "shard parity ok" in p.stdout
