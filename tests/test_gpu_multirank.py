"""Functional run of bench.py's multi-rank paths on one GPU: two ranks under
torchrun share cuda:0 over gloo (MCKG_BENCH_SHARED_GPU=1).  The C3 shards
(block ranges, MIN-all-reduced line table) and the C5 exchange (K3 partition,
all_to_all_single, K6 per owner) must report exactly what one rank reports."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(n, port):
    env = dict(os.environ, MCKG_BENCH_SHARED_GPU="1")
    args = ["bench.py", "--gpus", str(n), "--steps", "3", "--warmup", "3", "--blocks", "16384",
            "--c5-blocks", "2048", "--no-cpu", "--no-k1", "--e2e-blocks", "0"]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(port)] + args
    else:
        cmd = [sys.executable] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def test_two_ranks_report_what_one_rank_reports():
    one = _bench(1, 0)
    two = _bench(2, 29611)
    assert two["n_gpus"] == 2
    assert two["config"]["events"] == one["config"]["events"]
    assert two["config"]["reported_triples"] == one["config"]["reported_triples"]
    assert two["c5"]["races_reported"] == one["c5"]["races_reported"]
    assert two["c5"]["status"] == 0
