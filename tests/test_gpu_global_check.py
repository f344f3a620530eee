"""RunOptions::globalRaceCheck end to end: K1 logs every global access of a
grid, K6 finds the cross-block races, the host reports them as
"Possible race on global device memory detected at <file>:<line>." in
first-detection order (builder-defined).  With the option
off the run is the reference's own (goldens in tests/golden/global_check.json)."""
import json
import os

import pytest

from global_check_programs import PROGRAMS
from program_corpus import project

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "global_check.json")))


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_option_off_is_the_reference(name):
    from paper_1211_6193_b200 import checker
    r = checker.run_source(PROGRAMS[name][0], filename="g.cu")
    assert r["engine_error"] == ""
    got = project(r)
    for k, v in GOLD[name].items():
        assert got[k] == v, k


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_global_races_reported(name):
    from paper_1211_6193_b200 import checker
    src, lines = PROGRAMS[name]
    r = checker.run_source(src, filename="g.cu", global_race_check=True)
    assert r["engine_error"] == ""
    grace = [d for d in r["diags"] if "global device memory" in d["msg"]]
    assert [d["line"] for d in grace] == lines
    assert all(d["msg"] == f"Possible race on global device memory detected at g.cu:{d['line']}." and
               d["cat"] == "race" and d["sev"] == "warning" for d in grace)
    # everything else is unchanged; any diagnostic makes the exit code 1
    base = GOLD[name]
    assert r["output"] == base["output"] and r["steps"] == base["steps"]
    assert [d for d in r["diags"] if "global device memory" not in d["msg"]] == base["diags"]
    assert r["exit"] == (1 if lines and base["exit"] == 0 else base["exit"])


def test_full_size_c2_has_no_global_race():
    """The Fig. 1 reduction at 2^20 ints: blocks read disjoint inputs and
    write disjoint partial sums."""
    import gen_programs as gp
    from paper_1211_6193_b200 import checker
    r = checker.run_source(gp.scaled(1 << 20, 256), "c2.cu", step_limit=8_000_000_000, global_race_check=True)
    assert r["engine_error"] == ""
    assert r["exit"] == 0 and r["diags"] == []


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_conflicts_flagged_without_the_option(name):
    """With the option off the run stays the reference's, but a small grid
    with cross-block global conflicts -- whose values follow this engine's
    block order, not the reference's interleaving -- is named in
    RunResult::engineNote instead of diverging silently."""
    from paper_1211_6193_b200 import checker
    src, lines = PROGRAMS[name]
    for r in (checker.run_source(src, filename="g.cu"), checker.run(src, "g.cu")):
        assert r["engine_error"] == ""
        assert ("cross-block global-memory conflicts" in r["engine_note"]) == bool(lines), r["engine_note"]
        assert r["output"] == GOLD[name]["output"] and r["exit"] == GOLD[name]["exit"]


INFLIGHT = r"""#include <stdio.h>
__global__ void slow(int* g, int n) {
  int t = threadIdx.x, i, acc = t;
  for (i = 0; i < n; ++i) { acc = acc * 3 + i; }
  g[t] = acc %% 1000;
}
int main(void) {
  int *g, h[64];
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaMalloc(&g, 64 * sizeof(int));
  cudaMemset(g, 0, 64 * sizeof(int));
  slow<<<1, 64, 0, s1>>>(g, 40);
  %s
  cudaMemcpyAsync(h, g, 64 * sizeof(int), cudaMemcpyDeviceToHost, s2);
  cudaDeviceSynchronize();
  printf("%%d %%d\n", h[0], h[63]);
  return 0;
}
"""


def test_inflight_copy_reads_grid_as_of_its_sweep():
    """A copy on another stream reads a grid's output while the grid is in
    flight: the reference copies the bytes as of that sweep.  The grid ran at
    its dispatch, so the copy is rebuilt from the grid's write history (every
    write up to the copy's sweep over what it overwrote): "0 0", exactly the
    reference's own run.  Synchronised first, the copy sees the whole grid
    (reference: "-444 -893", exit 1, 74,537 steps)."""
    from paper_1211_6193_b200 import checker
    r = checker.run(INFLIGHT % "", "f.cu")
    assert r["output"] == "0 0\n" and r["exit"] == 1 and r["steps"] == 74530, r
    assert r["engine_note"] == ""
    r = checker.run(INFLIGHT % "cudaStreamSynchronize(s1);", "f.cu")
    assert r["engine_note"] == ""
    assert r["output"] == "-444 -893\n" and r["exit"] == 1 and r["steps"] == 74537


STAIRCASE = r"""#include <stdio.h>
__global__ void staircase(int* g) {
  int t = threadIdx.x, i, acc = 0;
  for (i = 0; i < t; ++i) { acc = acc + i; }
  g[t] = acc + 1;
}
int main(void) {
  int *g, h[32], i, spin = 0;
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaMalloc(&g, 32 * sizeof(int));
  cudaMemset(g, 0, 32 * sizeof(int));
  staircase<<<1, 32, 0, s1>>>(g);
  for (i = 0; i != %d; ++i) { spin = spin + i; }
  cudaMemcpyAsync(h, g, 32 * sizeof(int), cudaMemcpyDeviceToHost, s2);
  cudaDeviceSynchronize();
  for (i = 0; i != 32; ++i) printf("%%d ", h[i]);
  printf("\n%%d\n", spin);
  return 0;
}
"""
_TRI = [1, 1, 2, 4, 7, 11, 16, 22, 29, 37, 46, 56, 67, 79, 92, 106, 121, 137, 154, 172, 191, 211, 232, 254, 277,
        301, 326, 352, 379, 407, 436, 466]
# the reference's own runs (oracle/_ref, round robin): (host spin, steps, thread values copied, spin)
STAIR_GOLD = [(0, 14567, 0, 0), (10, 14807, 10, 45), (30, 15287, 29, 435), (60, 16007, 32, 1770),
              (200, 19367, 32, 19900)]


@pytest.mark.parametrize("k,steps,copied,spin", STAIR_GOLD)
def test_inflight_copy_sees_partial_grid(k, steps, copied, spin):
    """Threads finish at staggered sweeps; the host spins k iterations, then
    copies on another stream: the copy holds exactly the threads done by its
    sweep (reference goldens)."""
    from paper_1211_6193_b200 import checker
    r = checker.run(STAIRCASE % k, "m.cu")
    vals = _TRI[:copied] + [0] * (32 - copied)
    assert r["output"] == " ".join(map(str, vals)) + " \n%d\n" % spin, r["output"]
    assert r["exit"] == 0 and r["steps"] == steps and r["engine_note"] == ""
