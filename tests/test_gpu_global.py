"""K3/K6 (global-race extension, BASELINE config 5) against the CPU checker
oracle/global_detector.c: identical (byte, line) race sets and per-line
first-detection keys; parity with the reference itself is unpinned (the
reference has no global-race semantics)."""
import numpy as np
import pytest

import oracle_bind as ob

pytestmark = pytest.mark.gpu


MODES = {"dense": 256, "sparse": 128 | 256, "tile": 512, "tile_reread": 512 | 1024}


@pytest.fixture(autouse=True, params=list(MODES))
def k6_mode(request):
    """Every K6 route: the bucket pipeline in dense spans (warp per 2 KiB
    bucket, direct tables, the general kernel for what it hands back) and in
    sparse mode (hashed tables only, mckg_set_debug(128)), and the in-place
    tile path (pass 0 claim / foreign, pass 1 own words, the side list through
    the bucket pipeline), forced at any size by mckg_set_debug(512) and taken
    by default from 2^20 records -- its pass 1 from pass 0's per-record codes
    (single-block tiles) or re-reading every tile (mckg_set_debug(1024))."""
    from paper_1211_6193_b200 import _abi
    lib = _abi.load()
    lib.mckg_set_debug(MODES[request.param])
    yield request.param
    lib.mckg_set_debug(0)


def _dev(ev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(ev).view(np.int32).reshape(-1, 4).copy()).cuda()


def _detect(ev, addr_lo=0, capacity=None):
    from paper_1211_6193_b200 import global_race as gr
    t = _dev(ev)
    out = gr.GlobalOut(capacity if capacity is not None else 4 * len(ev) + 16)
    gr.detect(t, addr_lo, out.reset())
    races, n, lf, st = gr.fetch(out)
    order = np.lexsort((races["line"], races["addr"]))
    return races[order], n, lf, st


def _check(ev):
    races, n, lf, st = _detect(ev)
    rc, want, wn, wlf = ob.port_detect_global(ev)
    assert rc == 0 and st == 0
    assert n == wn
    assert np.array_equal(races["addr"], want["addr"]) and np.array_equal(races["line"], want["line"])
    assert np.array_equal(lf, wlf)
    return n


def test_gen_c5_matches_cpu_copy():
    from paper_1211_6193_b200 import global_race as gr
    ev = gr.gen_c5(3, 5, 40).cpu().numpy().view(ob.GACCESS_DTYPE).reshape(-1)
    assert np.array_equal(ev, ob.gen_c5(3, 5, 40))


def test_c5_sample():
    n = _check(ob.gen_c5(0, 64, 64))
    assert n > 0


def _random(seed, n=20000, nblocks=12, span=4096):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        length = int(rng.choice([1, 2, 4, 8]))
        addr = int(rng.integers(0, span)) if rng.random() < 0.7 else int(rng.integers(0, 64))
        rows.append(ob.make_gaccess(addr, length, rng.random() < 0.4, int(rng.integers(0, 64)),
                                    int(rng.integers(0, nblocks)), int(rng.integers(10, 40)),
                                    int(rng.integers(0, 500))))
    return np.array(rows, dtype=ob.GACCESS_DTYPE)


@pytest.mark.parametrize("seed", range(6))
def test_random_global_traces(seed):
    _check(_random(seed))


@pytest.mark.parametrize("seed", range(4))
def test_wide_sparse_traces(seed):
    """Records spread over a 2^36-byte window with clusters: empty buckets,
    crowded buckets, accesses crossing words and buckets."""
    rng = np.random.default_rng(100 + seed)
    rows = []
    centers = rng.integers(0, 1 << 36, size=8)
    for i in range(30000):
        c = int(centers[rng.integers(0, 8)])
        addr = c + int(rng.integers(0, 1 << int(rng.integers(4, 14))))
        rows.append(ob.make_gaccess(addr, int(rng.choice([1, 2, 4, 8])), rng.random() < 0.5,
                                    int(rng.integers(0, 32)), int(rng.integers(0, 6)), int(rng.integers(1, 60)),
                                    int(rng.integers(0, 3000))))
    _check(np.array(rows, dtype=ob.GACCESS_DTYPE))


def test_hot_word_many_blocks():
    """Thousands of blocks on one word: the global-memory tables path."""
    rows = [ob.make_gaccess(4096, 4, (i % 3) == 0, i % 64, i % 5000, 7 + (i % 3), i) for i in range(20000)]
    _check(np.array(rows, dtype=ob.GACCESS_DTYPE))


def test_two_owner_emulation_on_one_gpu():
    """The multi-GPU split: partition by owner, detect each part with its
    address base, union == single detection."""
    import torch
    from paper_1211_6193_b200 import global_race as gr
    ev = ob.gen_c5(0, 32, 32)
    space = 32 * 65536
    grouped, counts = gr.partition(_dev(ev), 2, space)
    torch.cuda.synchronize()
    c = counts.cpu().tolist()
    assert sum(c) == len(ev)
    allr, lfs = [], []
    off = 0
    for r in range(2):
        part = grouped[off:off + c[r]]
        off += c[r]
        lo, hi = gr.addr_range(r, 2, space)
        out = gr.GlobalOut(4 * len(ev))
        gr.detect(part, lo, out.reset())
        races, n, lf, st = gr.fetch(out)
        assert st == 0
        a = races["addr"]
        assert np.all((a >= lo) & (a < hi))
        allr += list(zip(a.tolist(), races["line"].tolist()))
        lfs.append(lf)
    rc, want, wn, wlf = ob.port_detect_global(ev)
    assert sorted(allr) == sorted(zip(want["addr"].tolist(), want["line"].tolist()))
    assert np.array_equal(np.minimum(lfs[0], lfs[1]), wlf)


def _tiled(nt, seed, shared_words, bids_per_tile=2, foreign=0.01, unaligned=0.0, overlap=False):
    """Block-clustered records, one TT-record tile per 32 KiB range: tile t
    writes/reads its range from `bids_per_tile` blocks; `shared_words` words
    per tile are touched by two of them (candidates inside a tile), a
    `foreign` fraction lands in the next range, `unaligned` cross words, and
    with `overlap` neighbouring tiles share half their range (contested
    buckets)."""
    rng = np.random.default_rng(seed)
    n = nt * 4096
    t = np.repeat(np.arange(nt, dtype=np.uint64), 4096)
    j = np.tile(np.arange(4096, dtype=np.uint64), nt)
    stride = 16384 if overlap else 32768
    addr = t * stride + (j * 8) % 32768
    bid = (t * bids_per_tile + (j % bids_per_tile)).astype(np.uint64)
    if shared_words:  # record k takes the word of record k ^ 1 (another block)
        k = rng.integers(0, 4096, size=(nt, shared_words)).astype(np.uint64)
        rows = (np.arange(nt, dtype=np.uint64)[:, None] * 4096 + k).reshape(-1)
        addr[rows] = addr[rows ^ np.uint64(1)]
    f = rng.random(n) < foreign
    addr[f] = ((t[f] + 1) % nt) * stride + (j[f] * 8) % 32768
    u = rng.random(n) < unaligned
    addr[u] += 2
    write = rng.random(n) < 0.5
    ln = np.full(n, 4, dtype=np.uint64)
    line = (100 + (j % 7)).astype(np.uint64)
    tid = j % 256
    a = (addr & 0xFFFFFFFFFF) | (ln << 40) | (write.astype(np.uint64) << 44) | (tid << 45) | ((line & 0xFF) << 56)
    ev = np.zeros(n, dtype=ob.GACCESS_DTYPE)
    ev["a"] = a
    ev["sweep"] = (j // 256).astype(np.uint32)
    ev["b"] = (bid & 0xFFFFFF).astype(np.uint32) | ((line >> 8).astype(np.uint32) << 24)
    return ev


@pytest.mark.parametrize("case", [
    dict(shared_words=0, bids_per_tile=1),                       # C5-like: own words race-free
    dict(shared_words=4, bids_per_tile=2, foreign=0.0),          # <= 32 candidates per tile
    dict(shared_words=200, bids_per_tile=2, foreign=0.0),        # > 32: the tile joins the side list
    dict(shared_words=8, bids_per_tile=3, foreign=0.02, unaligned=0.01),
    dict(shared_words=4, bids_per_tile=2, overlap=True),         # contested buckets
])
def test_block_clustered_traces(case):
    n = _check(_tiled(24, 7, **case))
    assert n >= 0


def test_single_and_multi_block_tiles_mixed():
    """One input whose tiles alternate between one block (pass 1 from pass
    0's codes, tile_mixed) and two blocks (listed for the re-reading pass),
    with foreign records between them, in-tile candidates, word-crossing
    records and a partial last tile (codes past its end are unused)."""
    ev = _tiled(40, 13, shared_words=5, bids_per_tile=2, foreign=0.02, unaligned=0.003)
    t = np.repeat(np.arange(40), 4096)
    single = (t % 2) == 0
    b = ev["b"] & 0xFFFFFF
    ev["b"][single] = (ev["b"][single] & 0xFF000000) | (b[single] & ~np.uint32(1))
    assert _check(ev[: 40 * 4096 - 1000]) > 0


def test_c5_two_million_records():
    """2^21 C5 records: the size at which the tile path is the default."""
    assert _check(ob.gen_c5(0, 512, 512)) > 0


def test_block_clustered_million_records():
    """2^20 block-clustered records with every tile-path hazard at once
    (in-tile candidates, foreign and word-crossing records, half-overlapping
    windows): the size at which the tile path is the default route."""
    ev = _tiled(256, 11, shared_words=6, bids_per_tile=2, foreign=0.02, unaligned=0.005)
    ev2 = _tiled(64, 12, shared_words=3, bids_per_tile=3, overlap=True)
    assert _check(np.concatenate([ev, ev2])) > 0


@pytest.mark.parametrize("k6_mode", ["tile"], indirect=True)
def test_c5_full_share_matches_port(k6_mode):
    """One GPU's full share of configs[4] (2^29 records, the default tile
    route) against the C checker, run address-partitioned over the host's
    cores: a byte lives in exactly one address range, so the per-range race
    sets are disjoint and the line table is their minimum."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    import psutil
    from paper_1211_6193_b200 import _abi
    from paper_1211_6193_b200 import global_race as gr
    if psutil.virtual_memory().available < (48 << 30):
        pytest.skip("needs ~48 GiB of host memory for the 8.6 GB trace and its partition")
    _abi.load().mckg_set_debug(0)  # the default route at this size
    blocks = 1 << 17
    ev_d = gr.gen_c5(0, blocks, blocks)
    out = gr.GlobalOut(ev_d.shape[0] // 8)
    gr.detect(ev_d, 0, out.reset())
    races, n, lf, st = gr.fetch(out)
    assert st == 0 and n == len(races)
    ev = ev_d.cpu().numpy().view(ob.GACCESS_DTYPE).reshape(-1)
    del ev_d, out
    addr = ev["a"] & np.uint64(0xFFFFFFFFFF)
    ln = (ev["a"] >> np.uint64(40)) & np.uint64(0xF)
    parts = 64
    shift = max(3, int(addr.max()).bit_length() - 6)  # 64 ranges, each a multiple of 8 bytes
    owner = (addr >> np.uint64(shift)).astype(np.uint8)
    assert np.array_equal(owner, ((addr + ln - np.uint64(1)) >> np.uint64(shift)).astype(np.uint8))
    del addr, ln
    order = np.argsort(owner, kind="stable")
    bounds = np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=parts))])
    del owner

    def check(p):
        part = np.ascontiguousarray(ev[order[bounds[p]:bounds[p + 1]]])
        if len(part) == 0:
            return np.zeros(0, dtype=ob.GRACE_DTYPE), 0, np.full(len(lf), ob.TS_NONE, dtype=np.uint64)
        rc, want, wn, wlf = ob.port_detect_global(part, capacity=4 * len(part) + 16)
        assert rc == 0
        return want, wn, wlf

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        res = list(pool.map(check, range(parts)))
    want = np.concatenate([r[0] for r in res])
    assert sum(r[1] for r in res) == n
    got = races[np.lexsort((races["line"], races["addr"]))]
    want = want[np.lexsort((want["line"], want["addr"]))]
    assert np.array_equal(got["addr"], want["addr"]) and np.array_equal(got["line"], want["line"])
    assert np.array_equal(lf, np.minimum.reduce([r[2] for r in res]))
