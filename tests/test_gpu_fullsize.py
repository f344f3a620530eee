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
