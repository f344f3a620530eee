"""Whole-program parity on the edge corpus (tests/edge_programs.py, goldens
from the reference itself in tests/golden/edge_programs.json): step limits
reached inside a grid, at the exact total and on the host
(Machine::run machine.cpp:1183-1191), and the capacity cases."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
EDGE = json.load(open(os.path.join(HERE, "golden", "edge_programs.json")))


@pytest.mark.parametrize("name", sorted(EDGE))
def test_edge_program(name):
    from paper_1211_6193_b200 import checker
    from program_corpus import project
    e = EDGE[name]
    ours = checker.run_source(e["src"], filename=e["fname"], step_limit=e["step_limit"])
    assert ours.get("engine_error", "") == "", ours.get("engine_error")
    got, want = project(ours), e["gold"]
    for k in want:
        assert got[k] == want[k], f"{name}: {k} differs:\n ours {got[k]!r}\n ref  {want[k]!r}"
