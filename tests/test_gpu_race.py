"""K2 (mckg_detect_shared) parity against the CPU oracle: bit-exact reported
triples (RaceState::reported, machine.hpp:91), bit-exact first-detection
timestamps per line (the Race diagnostic order, machine.cpp:41-46).

Every test runs on both K2 paths: the default two-kernel path (filter ->
per-block candidate lists -> exact_kernel, with the fused kernel redoing a
launch whose lists overflow) and the fused kernel alone (MCKG_DEBUG=32)."""
import numpy as np
import pytest

import oracle_bind as ob
from tracegen_py import random_trace

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["two_kernel", "fused"])
def k2_path(request, monkeypatch):
    if request.param == "fused":
        monkeypatch.setenv("MCKG_DEBUG", "32")
    else:
        monkeypatch.delenv("MCKG_DEBUG", raising=False)
    return request.param


def _gpu(ev, bs, shmem, capacity=None, obj_base=1, bid_base=0):
    import torch
    from paper_1211_6193_b200 import race
    if len(ev) == 0:
        dev_ev = torch.zeros((0, 4), dtype=torch.int32, device="cuda")
    else:
        dev_ev = torch.from_numpy(ev.view(np.int32).reshape(-1, 4).copy()).cuda()
    dev_bs = torch.from_numpy(bs.astype(np.int64)).cuda()
    return race.detect_shared(dev_ev, dev_bs, shmem, obj_base=obj_base, bid_base=bid_base,
                              capacity=capacity)


def _check(ev, bs, shmem, obj_base=1, bid_base=0):
    res = _gpu(ev, bs, shmem, obj_base=obj_base, bid_base=bid_base)
    rc, tri, n, lf = ob.port_detect(ob.make_trace(ev, bs, shmem, obj_base=obj_base,
                                                  bid_base=bid_base))
    assert rc == 0
    assert res.status == 0
    assert res.n_triples == n
    assert np.array_equal(res.triples, ob.sorted_triples(tri))
    assert np.array_equal(res.line_first, lf)
    return res, n


def test_c3_sample_matches_oracle():
    ev, bs = ob.gen_c3(0, 128)
    res, n = _check(ev, bs, ob.C3_SHMEM)
    assert n > 0 and res.race_lines == [101, 100] or res.race_lines == [100, 101]


def test_c3_shard_offsets():
    ev, bs = ob.gen_c3(1000, 64)
    _check(ev, bs, ob.C3_SHMEM, obj_base=77, bid_base=1000)


@pytest.mark.parametrize("seed", range(24))
def test_random_traces(seed):
    rng = np.random.default_rng(1000 + seed)
    ev, bs = random_trace(seed, n_blocks=int(rng.integers(1, 40)), threads=int(rng.integers(1, 65)),
                          shmem=int(rng.choice([8, 36, 64, 256, 1024])),
                          epochs=int(rng.integers(1, 6)), per_epoch=int(rng.integers(1, 200)),
                          p_write=float(rng.random()), hot=float(rng.random()),
                          empty_blocks=0.1)
    _check(ev, bs, _shm(seed))


def _shm(seed):
    rng = np.random.default_rng(1000 + seed)
    rng.integers(1, 40), rng.integers(1, 65)
    return int(rng.choice([8, 36, 64, 256, 1024]))


@pytest.mark.parametrize("kinds", [("int",), ("char",), ("long",), ("short",), ("mis",),
                                   ("int", "long"), ("char", "long", "mis")])
def test_granularities(kinds):
    ev, bs = random_trace(5, n_blocks=12, threads=40, shmem=128, epochs=4, per_epoch=150,
                          kinds=kinds, hot=0.5)
    _check(ev, bs, 128)


def test_many_epochs_and_big_blocks():
    ev, bs = random_trace(9, n_blocks=6, threads=1024, shmem=4096, epochs=60, per_epoch=70,
                          kinds=("int", "char"), hot=0.2)
    _check(ev, bs, 4096)


def test_single_thread_never_races():
    ev, bs = random_trace(3, n_blocks=8, threads=1, shmem=64, epochs=3, per_epoch=50)
    res, n = _check(ev, bs, 64)
    assert n == 0 and res.race_lines == []


def test_hot_word_all_threads():
    # every thread writes the same word in one epoch: tid 0 first, all others race
    rows = [ob.make_access(0, 4, True, t, 0, 17, t) for t in range(256)]
    ev = np.array(rows, dtype=ob.ACCESS_DTYPE)
    bs = np.array([0, len(ev)], dtype=np.uint64)
    res, n = _check(ev, bs, 4)
    assert n == 4 and res.race_lines == [17]


def test_empty_and_zero_event_blocks():
    ev = np.zeros(0, dtype=ob.ACCESS_DTYPE)
    bs = np.zeros(5, dtype=np.uint64)
    res, n = _check(ev, bs, 16)
    assert n == 0


def test_overflow_reports_full_count():
    ev, bs = ob.gen_c3(0, 16)
    res = _gpu(ev, bs, ob.C3_SHMEM, capacity=10)
    _, _, n, _ = ob.port_detect(ob.make_trace(ev, bs, ob.C3_SHMEM))
    assert res.status & 1 and res.n_triples == n and len(res.triples) == 10


def test_out_of_range_event_is_flagged():
    rows = [ob.make_access(62, 4, True, 0, 0, 5, 0), ob.make_access(0, 4, True, 1, 0, 5, 1)]
    ev = np.array(rows, dtype=ob.ACCESS_DTYPE)
    bs = np.array([0, 2], dtype=np.uint64)
    res = _gpu(ev, bs, 64)
    assert res.status & 2


def test_host_entry_point_matches_device():
    from paper_1211_6193_b200 import race
    ev, bs = ob.gen_c3(0, 300)
    hres = race.detect_shared_host(ev, bs, ob.C3_SHMEM)
    dres = _gpu(ev, bs, ob.C3_SHMEM)
    assert hres.status == 0
    assert np.array_equal(hres.triples, dres.triples)
    assert np.array_equal(hres.line_first, dres.line_first)


def test_c3_16m_events_matches_oracle():
    import torch
    from paper_1211_6193_b200 import race
    nb = 1 << 14
    ev, bs = race.gen_c3(0, nb)
    res = race.detect_shared(ev, bs, ob.C3_SHMEM)
    hev, hbs = ob.gen_c3(0, nb)
    rc, tri, n, lf = ob.port_detect(ob.make_trace(hev, hbs, ob.C3_SHMEM), nthreads=8)
    assert res.n_triples == n
    assert np.array_equal(res.triples, ob.sorted_triples(tri))
    assert np.array_equal(res.line_first, lf)
    del ev, bs
    torch.cuda.empty_cache()
