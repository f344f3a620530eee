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


def _bench(n, port, dump):
    env = dict(os.environ, MCKG_BENCH_SHARED_GPU="1")
    args = ["bench.py", "--gpus", str(n), "--steps", "3", "--warmup", "3", "--blocks", "16384",
            "--c5-blocks", "2048", "--no-cpu", "--no-k1", "--e2e-blocks", "0", "--dump", str(dump)]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(port)] + args
    else:
        cmd = [sys.executable] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def _sets(d, n):
    """Union of the ranks' result sets (C3 triples, C5 (addr, line) races) and
    their reduced line tables."""
    import numpy as np
    c3 = [np.load(os.path.join(d, f"c3_r{r}.npz")) for r in range(n)]
    c5 = [np.load(os.path.join(d, f"c5_r{r}.npz")) for r in range(n)]
    tri = np.concatenate([z["triples"] for z in c3])
    tri = tri[np.lexsort((tri["line"], tri["byte"], tri["obj"]))]
    races = np.concatenate([z["races"] for z in c5])
    races = races[np.lexsort((races["line"], races["addr"]))]
    return tri, c3[0]["line_first"], races[["addr", "line"]], c5[0]["line_first"], c3, c5


def test_two_ranks_report_what_one_rank_reports(tmp_path):
    import numpy as np
    one = _bench(1, 0, tmp_path / "one")
    two = _bench(2, 29611, tmp_path / "two")
    t1, lf1, r1, glf1, *_ = _sets(tmp_path / "one", 1)
    t2, lf2, r2, glf2, c3, c5 = _sets(tmp_path / "two", 2)
    # same reported sets, as sets (not counts), and the same report order
    assert len(t1) > 0 and np.array_equal(t1, t2)
    assert np.array_equal(lf1, lf2) and np.array_equal(c3[1]["line_first"], lf2)
    assert len(r1) > 0 and np.array_equal(r1, r2)
    assert np.array_equal(glf1, glf2) and np.array_equal(c5[1]["line_first"], glf2)
    assert two["n_gpus"] == 2
    assert two["config"]["events"] == one["config"]["events"]
    assert two["config"]["reported_triples"] == one["config"]["reported_triples"]
    assert two["c5"]["races_reported"] == one["c5"]["races_reported"]
    assert two["c5"]["status"] == 0
