"""The sharded (N-rank) engine path gives bit-identical prices to one rank.

Two ranks share the one GPU of the test box through the gloo backend:
collectives are host-staged, so no kernel of one rank waits on the other
(the NCCL path is the same code with the collectives on the device).
The reference's determinism contract across worker counts (cli.py:303-309)
is the bar: identical price and variance bits.
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(nproc, config, scale):
    args = ["bench.py", "--config", config, "--scale", str(scale), "--steps", "1", "--warmup", "0",
            "--no-cpu-baseline", "--no-fast-line", "--dist-backend", "gloo"]
    if nproc == 1:
        cmd = [sys.executable] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("config,scale", [("c5", 0.03), ("c2", 0.25), ("c2", 1.0), ("c1", 0.25)])
def test_two_ranks_bitwise_equal_to_one(config, scale):
    one = _run(1, config, scale)
    two = _run(2, config, scale)
    assert two["n_gpus"] == 2
    assert two["price"] == one["price"], (one["price"], two["price"])
    assert two["ci95"] == one["ci95"]
