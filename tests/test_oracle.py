"""CPU: pins the C restatement of the race detector / deadlock scan (oracle/,
the checker of the CUDA kernels) against the reference itself
(oracle/_ref/libmckref.so = Machine::recordAccess / clearEpoch of
/root/reference/proj, replayed block by block, SURVEY Appendix D probe6), and
against committed fixtures where the reference build is absent."""
import json
import os

import numpy as np
import pytest

import oracle_bind as ob
from conftest import requires_ref
from tracegen_py import random_trace

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "k2_fixtures.json")


def _port(ev, bs, shm, **kw):
    rc, tri, n, lf = ob.port_detect(ob.make_trace(ev, bs, shm, **kw))
    assert rc == 0
    return ob.sorted_triples(tri), n, lf


def _cases():
    cases = []
    for seed in range(40):
        rng = np.random.default_rng(77 + seed)
        shm = int(rng.choice([8, 36, 64, 256, 1024]))
        ev, bs = random_trace(seed, n_blocks=int(rng.integers(1, 12)), threads=int(rng.integers(1, 40)),
                              shmem=shm, epochs=int(rng.integers(1, 5)), per_epoch=int(rng.integers(1, 120)),
                              p_write=float(rng.random()), hot=float(rng.random()))
        cases.append((f"rand{seed}", ev, bs, shm))
    ev, bs = ob.gen_c3(0, 32)
    cases.append(("c3_32blocks", ev, bs, ob.C3_SHMEM))
    return cases


@requires_ref
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_port_matches_reference_replay(case):
    _, ev, bs, shm = case
    tri, n, lf = _port(ev, bs, shm)
    rc, rtri, rn, rlf = ob.ref_detect(ob.make_trace(ev, bs, shm))
    assert rc == 0
    assert n == rn
    assert np.array_equal(tri, ob.sorted_triples(rtri))
    assert np.array_equal(lf, rlf)


def test_port_matches_committed_fixtures():
    fx = json.load(open(FIX))
    for name, ev, bs, shm in _cases():
        f = fx[name]
        tri, n, lf = _port(ev, bs, shm)
        assert n == f["n"], name
        assert [list(map(int, t)) for t in tri.tolist()] == f["triples"], name
        got_lf = {str(l): int(lf[l]) for l in np.nonzero(lf != ob.TS_NONE)[0]}
        assert got_lf == f["line_first"], name


def test_c3_generator_is_deterministic_and_racy():
    ev, bs = ob.gen_c3(5, 4)
    ev2, _ = ob.gen_c3(5, 4)
    assert np.array_equal(ev, ev2)
    assert len(ev) == 4 * ob.C3_EVENTS_PER_BLOCK
    tri, n, _ = _port(ev, bs, ob.C3_SHMEM, obj_base=6, bid_base=5)
    assert n > 0


def test_deadlock_port_closed_form():
    # if (v % 2) __syncthreads();  -> waiting = odd-v tids, blocks with mixed parity deadlock
    rng = np.random.default_rng(3)
    nb, bd = 9, 40
    v = rng.integers(0, 100, size=(nb, bd))
    v[0] &= ~1
    v[1] |= 1
    arr = (v % 2).astype(np.uint32)
    wm, dl = ob.port_scan_stuck(arr.reshape(-1), nb, bd)
    words = (bd + 31) // 32
    for b in range(nb):
        odd = [t for t in range(bd) if v[b, t] % 2]
        mixed = 0 < len(odd) < bd
        assert (b in dl.tolist()) == mixed
        got = [t for t in range(bd) if (wm[b * words + t // 32] >> (t % 32)) & 1]
        assert got == (odd if mixed else [])


def test_trace_golden_is_the_reference():
    """tests/golden/traces.json was produced by the reference (oracle/_ref)."""
    import json
    import os
    if ob.ref() is None:
        pytest.skip("reference library not built here")
    from program_corpus import corpus
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "traces.json")))
    progs = {n: (f, s) for n, f, s in corpus()}
    for n in sorted(gold)[:10]:
        f, s = progs[n]
        assert ob.ref_run(s, f, capture=False, trace=True)["trace"] == gold[n]


def test_c3_chunked_replay_matches_whole_run():
    """tests/c3_parity.py (the full-size GPU parity leg) on a CPU-sized trace:
    the chunked reference replay reproduces a whole-trace detection."""
    import c3_parity
    nb = 3000
    ev, bs = ob.gen_c3(0, nb)
    rc, tri, n, lf = ob.port_detect(ob.make_trace(ev, bs, ob.C3_SHMEM), nthreads=4)
    assert rc == 0 and n > 0
    got = c3_parity.replay_full(ob.sorted_triples(tri), lf, nb, 4, chunk_blocks=1024)
    assert got["triples_equal"] and got["line_first_equal"], got
    assert got["reference_triples"] == n
    bad = ob.sorted_triples(tri).copy()
    bad["line"][len(bad) // 2] += 1
    got = c3_parity.replay_full(bad, lf, nb, 4, chunk_blocks=1024)
    assert not got["triples_equal"]
    part = c3_parity.replay_full(ob.sorted_triples(tri), lf, nb, 4, chunk_blocks=1024, max_blocks=1500)
    assert part["triples_equal"] and part["line_first_equal"] is None and part["checked_blocks"] == 1500
