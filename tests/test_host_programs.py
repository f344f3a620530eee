"""CPU parity of the host-thread interpreter and the step-exact IR against
the reference (golden Machine::run results in tests/golden/host_programs.json,
made by tests/make_golden.py): 400 random host programs plus handwritten
UB / runtime-API / stream cases, and frontend-error cases.  Device grids are
not involved; the value and step semantics checked here are the ones K1
shares (csrc/core.cuh, include/mck_ir.h)."""
import json
import os

import pytest

from program_corpus import FRONTEND_CASES, HOST_STEP_LIMIT, host_corpus, project

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "host_programs.json")))
CASES = {name: (fname, src) for name, fname, src in host_corpus()}


def _run(src, fname, **kw):
    from paper_1211_6193_b200 import checker
    return checker.run_source(src, filename=fname, **kw)


@pytest.mark.parametrize("name", sorted(CASES))
def test_host_program(name):
    fname, src = CASES[name]
    ours = _run(src, fname, step_limit=HOST_STEP_LIMIT)
    want = GOLD[name]
    if "frontend_error" in ours:
        assert want["exit"] == 2
        return
    assert ours.get("engine_error", "") == ""
    got = project(ours)
    for k in want:
        assert got[k] == want[k], f"{name}: {k} differs:\n ours {got[k]!r}\n ref  {want[k]!r}"


@pytest.mark.parametrize("name", sorted(FRONTEND_CASES))
def test_frontend_errors(name):
    ours = _run(FRONTEND_CASES[name], name + ".cu")
    want = GOLD["fe_" + name]
    assert ours["exit"] == 2
    assert ours["frontend_error"] == want["frontend_error"]
    assert ours["line"] == want["line"]


def test_launch_without_gpu_fails_loudly():
    """No CPU execution path for device code."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    src = "__global__ void k(void) { }\nint main(void) { k<<<1, 1>>>(); cudaDeviceSynchronize(); return 0; }\n"
    r = _run(src, "k.cu")
    assert "no CUDA device" in r["engine_error"] or r["engine_error"]


@pytest.mark.parametrize("name", sorted(CASES)[::20] + ["fe_" + n for n in sorted(FRONTEND_CASES)[:4]])
def test_result_record_abi_matches_json_abi(name):
    """mck_run / mck_result_* (records) return the same RunResult as mck_run_source (JSON)."""
    from paper_1211_6193_b200 import checker
    if name.startswith("fe_"):
        src, fname = FRONTEND_CASES[name[3:]], name[3:] + ".cu"
    else:
        fname, src = CASES[name]
    a = checker.run_source(src, filename=fname, step_limit=HOST_STEP_LIMIT)
    b = checker.run(src, filename=fname, step_limit=HOST_STEP_LIMIT)
    if "frontend_error" in a:
        assert b == {k: a[k] for k in ("frontend_error", "line", "exit")}
        return
    b["reported"] = [[int(t["obj"]), int(t["byte"]), int(t["line"])] for t in b["reported"]]
    for k in ("exit", "output", "steps", "stuck", "main_return", "engine_error", "diags", "stuck_reports",
              "report_text", "reported", "trace"):
        assert a[k] == b[k], k


def test_oracle_without_a_kernel_runs_on_the_host():
    """oracleRace of a host-only program: one schedule, nothing to explore."""
    from paper_1211_6193_b200 import checker
    r = checker.oracle_race("int main(void) { int x = 3; return x - 3; }\n")
    assert r == {"oracle_race": False, "detector_race": False, "interleavings": 1, "aborted": False, "error": ""}
    assert "frontend_error" in checker.oracle_race("int main(void) { return 0 }\n")
