"""Multi-GPU path through the C-ABI (NCCL min all-reduce + owner broadcast): the sharded
winner and assignment equal the single-GPU ones.  Runs tools/dist_check.py under torchrun;
skipped when fewer than two GPUs are visible.  -m gpu.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("k, batches", [(2, 0), (3, 0), (5, 0), (2, 3), (4, 0), (4, 2)])
def test_sharded_search_equals_single_gpu(k, batches):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(min(n, 2)),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "dist_check.py"),
           "--config", str(k), "--K", "4096", "--batches", str(batches)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    assert json.loads(line)["ok"] is True
