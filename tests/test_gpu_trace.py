"""--trace parity: the Machine::trace line stream --
stream dispatches (device.cpp:63, streams.cpp:49-61), barrier rules
(device.cpp:163-195) and grid completion (device.cpp:215) -- regenerated from
the B200 run (host timeline + per-thread barrier arrival sweeps recorded by
K1) must equal the reference's, line for line (tests/golden/traces.json,
tests/make_trace_golden.py)."""
import json
import os

import pytest

from program_corpus import corpus

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "traces.json")))
CORPUS = {name: (fname, src) for name, fname, src in corpus()}


@pytest.mark.parametrize("name", sorted(GOLD))
def test_trace_matches_reference(name):
    from paper_1211_6193_b200 import checker
    fname, src = CORPUS[name]
    r = checker.run_source(src, filename=fname, trace=True)
    assert r.get("engine_error", "") == "", r.get("engine_error")
    got, want = r["trace"], GOLD[name]
    for i, (a, b) in enumerate(zip(got, want)):
        assert a == b, f"{name}: line {i} differs:\n ours {a!r}\n ref  {b!r}"
    assert len(got) == len(want), (name, len(got), len(want))
