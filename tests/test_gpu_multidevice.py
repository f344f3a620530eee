"""Multi-device K1: every grid's blocks are split into contiguous ranges over
several devices (global memory replicated, merged after the grid).  On one
GPU the split runs over *virtual* devices (the same ordinal repeated), which
exercises the whole split / merge path; results must stay identical to the
reference's golden runs (tests/golden/programs.json)."""
import json
import os

import pytest

from program_corpus import corpus, project

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "programs.json")))
CORPUS = {name: (fname, src) for name, fname, src in corpus()}
ALL = sorted(n for n in CORPUS if n in GOLD)
SUBSET = [n for n in ALL if not n[-1].isdigit() or n.endswith(("0", "7"))]


def _check(name, devices):
    from paper_1211_6193_b200 import checker
    fname, src = CORPUS[name]
    ours = checker.run_source(src, filename=fname, devices=devices)
    assert ours.get("engine_error", "") == "", ours.get("engine_error")
    got, want = project(ours), GOLD[name]
    for k in want:
        assert got[k] == want[k], f"{name} on {devices}: {k} differs:\n ours {got[k]!r}\n ref  {want[k]!r}"


@pytest.mark.parametrize("name", ALL)
def test_two_virtual_devices(name):
    _check(name, [0, 0])


@pytest.mark.parametrize("name", SUBSET)
def test_three_virtual_devices(name):
    _check(name, [0, 0, 0])


def test_physical_devices():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("one GPU visible")
    for name in SUBSET[:50]:
        _check(name, list(range(min(n, 8))))
