"""The exhaustive-interleaving oracle on the GPU (mck::oracleRace /
mck_oracle) against the reference's own oracleRace (goldens in
tests/golden/oracle.json, tests/make_oracle_golden.py): the number of
interleavings, the ground-truth race verdict (traceHasRace,
oracle.cpp:47-71), the shadow detector's verdict and the abort reasons.  Then
past the reference's bounds: four threads and 6.35 million schedules."""
import json
import os

import pytest

from oracle_programs import PROGRAMS

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "oracle.json")))


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_oracle_matches_reference(name):
    from paper_1211_6193_b200 import checker
    src, o = PROGRAMS[name]
    got = checker.oracle_race(src, "o.cu", max_interleavings=o["max_interleavings"], max_threads=o["max_threads"],
                              max_accesses_per_thread=o["max_accesses"])
    want = GOLD[name]
    assert got["aborted"] == want["aborted"] and got["error"] == want["error"], got
    assert got["interleavings"] == want["interleavings"], got
    if not want["aborted"]:  # after an abort the verdicts depend on the exploration order
        assert got["oracle_race"] == want["oracle_race"] and got["detector_race"] == want["detector_race"], got


def test_lifted_bound_four_threads():
    """Four threads, two visible steps per thread per barrier phase:
    (8! / 2!^4)^2 = 6,350,400 schedules, none racing."""
    from paper_1211_6193_b200 import checker
    src, _ = PROGRAMS["four_threads"]
    got = checker.oracle_race(src, "o.cu", max_interleavings=100_000_000, max_threads=8)
    assert not got["aborted"], got
    assert got["interleavings"] == 2520 ** 2
    assert not got["oracle_race"] and not got["detector_race"]


def test_lifted_bound_racy_four_threads():
    """The same shape without the barrier: 8!/(2!^4)... every schedule of
    four threads' 4 visible steps, C(16; 4,4,4,4) = 63,063,000 leaves, racing."""
    from paper_1211_6193_b200 import checker
    src = PROGRAMS["four_threads"][0].replace("  __syncthreads();\n", "")
    got = checker.oracle_race(src, "o.cu", max_interleavings=100_000_000, max_threads=8)
    assert not got["aborted"], got
    assert got["interleavings"] == 63063000
    assert got["oracle_race"] and got["detector_race"]
