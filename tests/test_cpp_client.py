"""Builds tests/cpp/test_client.cpp -- a reference-style C++ client of
include/mck/checker.hpp (a subset of the reference's own unit tests plus the
hooks, scanStuck and the batched recordAccess/clearEpoch) -- against
libmckg.so and runs it: the host-only cases here, all cases on the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1211_6193_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_client")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_client.cpp"), "-o", exe, "-L" + PKG, "-lmckg",
                    "-Wl,-rpath," + PKG], check=True)
    return exe


def _run(exe, *args):
    env = dict(os.environ, MCK_CORPUS_DIR=os.path.join(ROOT, "tests", "golden"))
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout + out.stderr
    return out.stdout


def test_cpp_client_host_cases(tmp_path):
    print(_run(_build(tmp_path), "--no-gpu"))


@pytest.mark.gpu
def test_cpp_client_all_cases(tmp_path):
    out = _run(_build(tmp_path))
    assert " 0 skipped" in out
