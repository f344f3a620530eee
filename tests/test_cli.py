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
        # driver.cpp:152-158: header, the stuck reports, then the configuration dump
        text = (tmp_path / "report.txt").read_text()
        head = "stuck-state report for " + fname + "\n\n" + want["report_text"] + "\nfinal configuration:\n"
        assert text.startswith(head)


@needs_cli
def test_cli_arch_file_and_corpus(tmp_path):
    """--arch (loadArchFile, driver.cpp:39-84) and --run-corpus (runCorpus,
    driver.cpp:280-340) on host-only fixtures (no GPU needed)."""
    (tmp_path / "arch.txt").write_text("# B200-ish\nwarpSize = 32\nmaxThreadsPerBlock = 512\n")
    src = "int main(void) { return 0; }\n"
    out = _run(tmp_path, "a.cu", src, "--arch", "arch.txt")
    assert out.returncode == 0, out.stderr
    (tmp_path / "bad.txt").write_text("warpSize = x\n")
    out = _run(tmp_path, "a.cu", src, "--arch", "bad.txt")
    assert out.returncode == 2 and "bad.txt:1: 'x' is not an integer" in out.stderr
    corp = tmp_path / "corpus"
    corp.mkdir()
    (corp / "ok.cu").write_text('#include <stdio.h>\nint main(void) { printf("hi %d\\n", 7); return 0; }\n')
    (corp / "ok.expect").write_text("exit 0\nstdout<<EOF\nhi 7\nEOF\n")
    (corp / "ret.cu").write_text("int main(void) { return 5; }\n")
    (corp / "ret.expect").write_text("exit 4\n")
    (corp / "nosidecar.cu").write_text("int main(void) { return 0; }\n")
    r = subprocess.run([MCKB, "--run-corpus", str(corp)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1
    lines = r.stdout.splitlines()
    assert lines[0].startswith("FAIL nosidecar.cu (missing sidecar")
    assert lines[1] == "PASS ok.cu"
    assert lines[2] == "FAIL ret.cu (exit code 5, expected 4)"
    assert lines[3] == "1 passed, 2 failed"
