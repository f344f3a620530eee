"""tools/mckb -- the C++ driver over include/mck/checker.hpp (the reference CLI's
checking path): stdout, "cudak: " diagnostic lines, exit codes and the stuck
report file, against the reference goldens."""
import json
import os
import subprocess

import pytest

from program_corpus import HOST_STEP_LIMIT, corpus, host_corpus

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
MCKB = os.path.join(ROOT, "tools", "mckb")
HOST_GOLD = json.load(open(os.path.join(HERE, "golden", "host_programs.json")))
GOLD = json.load(open(os.path.join(HERE, "golden", "programs.json")))

needs_cli = pytest.mark.skipif(not os.path.exists(MCKB), reason="tools/mckb not built")


def _run(tmp_path, fname, src, *args):
    # the diagnostics name the file as given: run from tmp_path with the bare name
    (tmp_path / fname).write_text(src)
    return subprocess.run([MCKB, *args, fname], cwd=tmp_path, capture_output=True, text=True, timeout=120)


@needs_cli
@pytest.mark.parametrize("name", ["host3", "host7", "host11", "dead_pointer", "api_errors", "memcpy_roundtrip",
                                  "streams_events", "uninit"])
def test_cli_host_programs(tmp_path, name):
    cases = {n: (f, s) for n, f, s in host_corpus()}
    fname, src = cases[name]
    out = _run(tmp_path, fname, src, "--step-limit", str(HOST_STEP_LIMIT))
    want = HOST_GOLD[name]
    assert out.returncode == want["exit"]
    if want["exit"] == 2:  # frontend error: no run
        assert "error" in out.stderr
        return
    assert out.stdout == want["output"]
    assert out.stderr == "".join("cudak: " + d["msg"] + "\n" for d in want["diags"])


@needs_cli
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fig1", "fig1_race", "fig1_deadlock"])
def test_cli_fig1_family(tmp_path, name):
    cases = {n: (f, s) for n, f, s in corpus()}
    fname, src = cases[name]
    out = _run(tmp_path, fname, src, "--report", "report.txt")
    want = GOLD[name]
    assert out.returncode == want["exit"]
    assert out.stdout == want["output"]
    assert out.stderr == "".join("cudak: " + d["msg"] + "\n" for d in want["diags"])
    if want["exit"] == 3:
        assert (tmp_path / "report.txt").read_text() == want["report_text"]
