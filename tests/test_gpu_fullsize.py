"""BASELINE configs[1] at FULL size (2^24 ints, 65536 blocks x 256 threads)
through the whole checker, clean and racy, against goldens derived from
reference runs (tests/make_c2_golden.py: affine step counts, the period-25
input, the per-block reported pattern): exit code, OUTPUT, total steps, the
diagnostic list and all 33,292,288 RaceState::reported triples of the racy
run."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "c2_full.json")))


@pytest.mark.parametrize("variant", ["clean", "racy"])
def test_c2_full_size(variant):
    import gen_programs as gp
    from paper_1211_6193_b200 import checker
    g = GOLD[variant]
    nb, nt = GOLD["blocks"], GOLD["threads"]
    r = checker.run(gp.scaled(nb * nt, nt, racy=variant == "racy"), "c2.cu", step_limit=8_000_000_000)
    assert r["engine_error"] == ""
    assert r["exit"] == g["exit"]
    assert r["output"] == g["output"]
    assert r["steps"] == g["steps"]
    assert r["diags"] == g["diags"]
    rep = r["reported"]
    if variant == "clean":
        assert len(rep) == 0
        return
    assert len(rep) == g["reported"] == 33292288
    pat = np.array(g["block_pattern"], dtype=np.int64)
    k = len(pat)
    assert np.array_equal(rep["obj"].astype(np.int64), np.repeat(np.arange(nb, dtype=np.int64) + g["first_object"], k))
    assert np.array_equal(rep["byte"].astype(np.int64).reshape(nb, k), np.broadcast_to(pat[:, 0], (nb, k)))
    assert np.array_equal(rep["line"].astype(np.int64).reshape(nb, k), np.broadcast_to(pat[:, 1], (nb, k)))


def test_c4_full_size():
    """BASELINE configs[3] at full size (2^16 blocks x 1024 threads, the
    divergent-barrier sweep) against its closed form (a block
    deadlocks iff its threads' barrier counts differ; waiting = the threads
    with more calls, missing = the rest -- validated against the reference
    on 80 runs): exit 3, every deadlocked block in ascending order with its
    waiting / missing counts, and the full lists of the first 256."""
    import gen_programs as gp
    from paper_1211_6193_b200 import checker
    nb, nt = 1 << 16, 1024
    r = checker.run(gp.divergent_barrier_gen(nb, nt, 0), "c4.cu", step_limit=8_000_000_000, stuck_lists=256)
    assert r["engine_error"] == ""
    assert r["exit"] == 3 and r["stuck"]
    i = np.arange(nb * nt, dtype=np.int64).reshape(nb, nt)
    b = np.arange(nb, dtype=np.int64)[:, None]
    v = np.where(b % 3 == 0, 2 * i, np.where(b % 3 == 1, 2 * i + 1, (i * 3 + b) % 7))
    odd = (v % 2) == 1
    mixed = odd.any(1) & ~odd.all(1)
    want = np.nonzero(mixed)[0]
    bar = [s for s in r["stuck_reports"] if s["kind"] == "barrier"]
    assert [s["bid"] for s in bar] == want.tolist()
    nodd = odd.sum(1)
    assert [s["n_waiting"] for s in bar] == nodd[want].tolist()
    assert [s["n_missing"] for s in bar] == (nt - nodd[want]).tolist()
    for s in bar[:256]:
        assert s["waiting"] == np.nonzero(odd[s["bid"]])[0].tolist()
        assert s["missing"] == np.nonzero(~odd[s["bid"]])[0].tolist()
