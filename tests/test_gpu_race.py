"""K2 (mckg_detect_shared) parity against the reference: bit-exact reported
triples (RaceState::reported, machine.hpp:91), bit-exact first-detection
timestamps per line (the Race diagnostic order, machine.cpp:41-46).

Every test runs on both K2 paths: the default path (fast_kernel, one warp per
trace-mode block, with the general kernel redoing the blocks it hands back)
and the general kernel alone (mckg_set_debug(32))."""
import numpy as np
import pytest

import oracle_bind as ob
from tracegen_py import random_trace

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["fast", "general"])
def k2_path(request):
    from paper_1211_6193_b200 import _abi
    lib = _abi.load()
    lib.mckg_set_debug(32 if request.param == "general" else 0)
    yield request.param
    lib.mckg_set_debug(0)


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


def _oracle(trace, nthreads=1, capacity=None):
    """The reference's own recordAccess/clearEpoch replay (oracle/_ref, built
    here and shipped to the GPU box); the C restatement only where it is absent."""
    if ob.ref() is not None:
        return ob.ref_detect(trace, nthreads=nthreads, capacity=capacity)
    return ob.port_detect(trace, nthreads=nthreads, capacity=capacity)


def _check(ev, bs, shmem, obj_base=1, bid_base=0):
    res = _gpu(ev, bs, shmem, obj_base=obj_base, bid_base=bid_base)
    rc, tri, n, lf = _oracle(ob.make_trace(ev, bs, shmem, obj_base=obj_base, bid_base=bid_base))
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
    _, _, n, _ = _oracle(ob.make_trace(ev, bs, ob.C3_SHMEM))
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
    rc, tri, n, lf = _oracle(ob.make_trace(hev, hbs, ob.C3_SHMEM), nthreads=8)
    assert res.n_triples == n
    assert np.array_equal(res.triples, ob.sorted_triples(tri))
    assert np.array_equal(res.line_first, lf)
    del ev, bs
    torch.cuda.empty_cache()


def test_reference_present_on_gpu_box():
    """oracle/_ref travels with the snapshot: parity here is against the reference."""
    assert ob.ref() is not None


def test_c3_full_size_matches_reference(k2_path):
    """The headline workload at full size: 2^30 events, 2^20 blocks, every
    reported triple and every line's first-detection timestamp compared with
    the reference replay (chunked over all host cores, tests/c3_parity.py)."""
    if k2_path == "general":
        pytest.skip("full size runs once, on the default path")
    import os
    import torch
    import c3_parity
    from paper_1211_6193_b200 import race
    nb = 1 << 20
    ev, bs = race.gen_c3(0, nb)
    res = race.detect_shared(ev, bs, ob.C3_SHMEM, capacity=nb * 64, max_block_events=1024)
    del ev, bs
    torch.cuda.empty_cache()
    assert res.status == 0
    got = c3_parity.replay_full(res.triples, res.line_first, nb, len(os.sched_getaffinity(0)))
    assert got["triples_equal"], got["mismatch"]
    assert got["line_first_equal"]
    assert got["reference_triples"] == res.n_triples == 31773232


def _mixed_blocks(seed, nb=80):
    """Full 1024-record C3 blocks, every fifth one left as is and the others
    mutated so that the fast path must hand them to the general kernel: a hot
    word (> 32 candidates), a third epoch, a 1-byte access, a 2-byte access."""
    ev, bs = ob.gen_c3(seed * 1000, nb)
    ev = ev.copy()
    rng = np.random.default_rng(seed)
    for b in range(nb):
        blk = ev[b * 1024:(b + 1) * 1024]
        kind = b % 5
        if kind == 1:  # 64 threads of epoch 0 write slot 0
            for i in rng.choice(512, 64, replace=False):
                blk["w0"][i] = (int(blk["w0"][i]) & 0xFFF00000) | (1 << 24)
        elif kind == 2:  # the last 100 records move to a third epoch
            e = (blk["w1"][-1] >> 11) + 1
            blk["w1"][-100:] = (blk["w1"][-100:] & np.uint32(0x7FF)) | np.uint32(int(e) << 11)
        elif kind == 3:  # one aligned 1-byte access
            i = int(rng.integers(1024))
            blk["w0"][i] = (int(blk["w0"][i]) & 0xFF0FFFFF) | (1 << 20)
        elif kind == 4:  # one 2-byte access in the upper half of a word
            i = int(rng.integers(1024))
            blk["w0"][i] = ((int(blk["w0"][i]) & 0xFF0FFFFF) | (2 << 20)) + 2
        ev[b * 1024:(b + 1) * 1024] = blk
    return ev, bs


@pytest.mark.parametrize("seed", range(4))
def test_fast_path_hands_back_other_blocks(seed):
    """Blocks outside the fast path's shape are redone by the general kernel
    and the whole result still equals the reference's."""
    ev, bs = _mixed_blocks(seed)
    res, n = _check(ev, bs, ob.C3_SHMEM, obj_base=5, bid_base=seed * 1000)
    assert n > 0


def test_unsorted_epochs_are_flagged():
    ev, bs = ob.gen_c3(0, 8)
    ev = ev.copy()
    blk = ev[3 * 1024:4 * 1024]
    blk["w1"][[10, 900]] = blk["w1"][[900, 10]]  # an epoch-1 record before an epoch-0 one
    ev[3 * 1024:4 * 1024] = blk
    res = _gpu(ev, bs, ob.C3_SHMEM)
    assert res.status & 4


def test_oversize_blocks_8192_events():
    """Blocks beyond the kernels' 4096-record staging (the reference bounds
    neither): 8192-event blocks beside ordinary ones, through the oversize
    route, against the reference."""
    ev1, bs1 = random_trace(11, n_blocks=3, threads=512, shmem=2048, epochs=3, per_epoch=2800,
                            kinds=("int", "char", "long"), hot=0.3)
    ev2, bs2 = random_trace(12, n_blocks=4, threads=64, shmem=2048, epochs=2, per_epoch=100)
    ev = np.concatenate([ev1, ev2])
    bs = np.concatenate([bs1, bs2[1:] + bs1[-1]]).astype(np.uint64)
    assert np.diff(bs.astype(np.int64)).max() > 4096
    res, n = _check(ev, bs, 2048)
    assert n > 0


def test_oversize_shared_object():
    """A 256 KiB shared object: past the on-chip filter, every block takes
    the oversize route."""
    ev, bs = random_trace(13, n_blocks=5, threads=96, shmem=262144, epochs=2, per_epoch=400,
                          kinds=("int", "long"), hot=0.6)
    res, n = _check(ev, bs, 262144)
    assert n > 0


@pytest.mark.parametrize("n", [1, 2, 4095, 4097, 3_000_000])
def test_sort_triples_hand_written_radix(n):
    """mckg_sort_triples (the hand-written radix sort + unique of sort.cu):
    std::set order and the distinct set, against numpy."""
    import ctypes
    import torch
    from paper_1211_6193_b200 import _abi, race
    rng = np.random.default_rng(n)
    tri = np.zeros(n, dtype=ob.TRIPLE_DTYPE)
    tri["obj"] = 7 + rng.integers(0, 1 << 12, n)
    tri["byte"] = rng.integers(0, 1 << 20, n)
    tri["line"] = rng.integers(0, 1 << 16, n)
    tri[n // 2:] = tri[: n - n // 2]  # duplicates
    dev = torch.from_numpy(tri.view(np.int32).reshape(-1, 3).copy()).cuda()
    nu = torch.zeros(1, dtype=torch.int64, device="cuda")
    lib = _abi.load()
    _abi.check(lib.mckg_sort_triples(ctypes.c_void_p(dev.data_ptr()), n, 7, ctypes.c_void_p(nu.data_ptr()),
                                     race._stream_handle(None)), "mckg_sort_triples")
    torch.cuda.synchronize()
    want = np.unique(tri[np.lexsort((tri["line"], tri["byte"], tri["obj"]))])
    k = int(nu.item())
    got = dev[:k].cpu().numpy().view(ob.TRIPLE_DTYPE).reshape(-1)
    assert k == len(want) and np.array_equal(got, want)
