"""bench.py's N>1 paths end to end (torchrun, 2 and 4 ranks) on the one GPU the tests get:
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


@pytest.mark.parametrize("world,mode", [(2, "qdir"), (2, "exact"), (4, "qdir"), (4, "exact")])
def test_bench_multi_ranks(world, mode):
    """The split-step graphs (score graph -> gather -> apply graph) replayed on every rank;
    replicas bit-identical after the run."""
    env = dict(os.environ, ZO_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(world),
           "--model", "opt-125m", "--steps", "4", "--warmup", "3", "--mode", mode, "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == world and line["replicas_identical"] is True
    assert line["scaling"] == ("weak" if mode == "qdir" else "strong")
    assert line["config"]["parallelism"] == (f"qdir{world}" if mode == "qdir" else f"exact-dp{world}")
    # every timed step replays the captured score / apply halves (two graph launches)
    assert line["split_graphs"]["score_kernels"] > 10 and line["split_graphs"]["apply_kernels"] >= 2
    # end to end at N = 2: host batches per rank, the gathered coefficients read back every step
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] >= 32
