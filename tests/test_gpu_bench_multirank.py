"""bench.py's N>1 paths end to end (torchrun, 2 ranks) on the one GPU the tests get:
ZO_BENCH_SAME_DEVICE=1 puts both ranks on cuda:0 and exchanges through gloo, so this
checks the launch/exchange/timing flow and that every replica ends bit-identical
(q-direction and exact modes) -- not the NCCL performance."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["qdir", "exact"])
def test_bench_two_ranks(mode):
    env = dict(os.environ, ZO_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--model", "opt-125m",
           "--steps", "4", "--warmup", "3", "--mode", mode, "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["replicas_identical"] is True
    assert line["scaling"] == ("weak" if mode == "qdir" else "strong")
    assert line["config"]["parallelism"] == ("qdir2" if mode == "qdir" else "exact-dp2")
    # end to end at N = 2: host batches per rank, the gathered coefficients read back every step
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] >= 32
