"""K1 sharded over ranks (one process per GPU): rank r runs
blocks [gridDim*r/W, gridDim*(r+1)/W) of every grid; the written global bytes
are combined by an all-reduce(MAX) over the written range and the partial
reports are all-gathered, so every rank continues the host program with the
same memory.  On a one-GPU box the ranks share cuda:0 and use the host
transport (gloo); with >= 2 GPUs the NCCL transport is exercised too.
Results must equal the reference's golden runs."""
import json
import os
import subprocess
import sys

import pytest

from program_corpus import corpus

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = json.load(open(os.path.join(HERE, "golden", "programs.json")))
NAMES = sorted(n for n, _, _ in corpus() if n in GOLD)
PICK = [n for n in NAMES if not n[-1].isdigit() or n.endswith(("3", "8"))]


def _run(world, transport, names, port, tmp_path):
    out = tmp_path / f"r{world}{transport}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "rank_worker.py"), str(out), transport, ",".join(names)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.load(open(out))


def _compare(res):
    bad = []
    for n, got in res.items():
        assert got["engine_error"] == "", (n, got["engine_error"])
        for k, v in GOLD[n].items():
            if got[k] != v:
                bad.append((n, k, got[k], v))
    assert not bad, bad[:3]


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_share_one_gpu_host_transport(world, tmp_path):
    _compare(_run(world, "host", PICK, 29630 + world, tmp_path))


def test_ranks_nccl_transport(tmp_path):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("NCCL transport needs one GPU per rank")
    _compare(_run(min(n, 4), "nccl", PICK, 29640, tmp_path))


def test_nccl_exchange_path_one_rank(monkeypatch):
    """MCKG_K1_FORCE_EXCHANGE=1 runs the full NCCL exchange (dirty-range
    all-reduce, packed-byte all-reduce(MAX), result all-gather) on a
    one-rank communicator: the NCCL code path on a one-GPU box."""
    from paper_1211_6193_b200 import checker
    from program_corpus import project
    monkeypatch.setenv("MCKG_K1_FORCE_EXCHANGE", "1")
    progs = {n: (f, s) for n, f, s in corpus()}
    res = {}
    for n in PICK[::6]:  # a communicator per run (~1 s of NCCL setup each)
        fname, src = progs[n]
        r = checker.run_source(src, filename=fname)
        res[n] = dict(project(r), engine_error=r.get("engine_error", ""))
    _compare(res)
