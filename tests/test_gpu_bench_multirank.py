"""bench.py's multi-rank flow (torchrun, label shards, the peer grad_X
all-reduce with its warm-up checks, max-over-ranks timing, one JSON line from
rank 0) on the one-GPU box: XMC_BENCH_ONE_DEVICE=1 puts both ranks on cuda:0
with gloo.  Timings of such a run are meaningless (the ranks time-slice); the
test checks the path taken and the line's contract keys."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("peer", ["1", "0"])
def test_bench_two_ranks_one_device(peer):
    env = dict(os.environ, XMC_BENCH_ONE_DEVICE="1", XMC_PEER=peer)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--no-cpu", "--e2e-steps", "1", "--labels", "400000"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    for key in ("e2e", "roofline", "clocks", "gpu_launches"):
        assert key in d
    want = "peer memory" if peer == "1" else "gloo all_reduce"
    assert d["grad_x_allreduce"].startswith(want), d["grad_x_allreduce"]
