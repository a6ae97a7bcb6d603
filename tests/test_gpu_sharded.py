"""KV-head-sharded session end to end on one GPU: two ranks (gloo, both on
cuda:0) vs the unsharded session — identical tokens and records, across
partial-cache refreshes (the score exchange) and every layer's attention-output
all-gather (parallel.py; the NCCL path on N GPUs runs the same code)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--bf16"]], ids=["fp32-dh32", "bf16-dh128"])
def test_two_rank_sharded_session_equals_unsharded(extra):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tools", "mp_sharded_check.py"), *extra],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "identical to unsharded: True" in r.stdout, r.stdout[-2000:]
