"""CPU, world_size 2 over gloo: the multi-rank plumbing of the global-race
extension (paper_1211_6193_b200/global_race.py) -- block sharding, address-range
ownership, count exchange + all_to_all_single of 16-byte records, MIN
all-reduce of the line table.  Each rank runs the CPU checker (oracle) on the
records it owns; the union must equal a single-process run over all records,
which is what the GPU path (NCCL + K6) relies on."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, n_total, space, q):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import oracle_bind as ob
    from paper_1211_6193_b200 import global_race as gr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        b0, b1 = gr.shard(n_total, rank, ws)
        ev = ob.gen_c5(b0, b1 - b0, n_total)
        owner = gr.owner_of(ev["a"] & np.uint64(0xFFFFFFFFFF), ws, space)
        order = np.argsort(owner, kind="stable")
        grouped = np.ascontiguousarray(ev[order])
        counts = torch.tensor(np.bincount(owner.astype(np.int64), minlength=ws), dtype=torch.int64)
        t = torch.from_numpy(grouped.view(np.int32).reshape(-1, 4).copy())
        got = gr.exchange(t, counts)
        recv = got.numpy().view(ob.GACCESS_DTYPE).reshape(-1)
        lo, hi = gr.addr_range(rank, ws, space)
        addrs = recv["a"] & np.uint64(0xFFFFFFFFFF)
        assert np.all((addrs >= lo) & (addrs < hi)), "records delivered to their owner"
        rc, races, n, lf = ob.port_detect_global(recv)
        assert rc == 0
        lft = torch.from_numpy(lf.view(np.int64).copy())
        gr.min_allreduce_u64(lft)
        allr = [None] * ws
        dist.all_gather_object(allr, races.tolist())
        if rank == 0:
            q.put((sorted(x for r in allr for x in r), lft.numpy().view(np.uint64).tolist(), len(recv)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2])
def test_c5_exchange_matches_single_process(ws):
    import oracle_bind as ob
    n_total, space = 24, 24 * 65536
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, n_total, space, q)) for r in range(ws)]
    for p in procs:
        p.start()
    races, lf, _ = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ev = ob.gen_c5(0, n_total, n_total)
    rc, want, n, wlf = ob.port_detect_global(ev)
    assert rc == 0 and n > 0
    assert races == sorted(want.tolist())
    assert lf == wlf.tolist()


def test_owner_ranges_partition_the_space():
    from paper_1211_6193_b200 import global_race as gr
    space = 1 << 20
    for ws in (1, 2, 3, 8):
        addrs = np.arange(0, space, 97, dtype=np.uint64)
        own = gr.owner_of(addrs, ws, space)
        for r in range(ws):
            lo, hi = gr.addr_range(r, ws, space)
            sel = addrs[own == r]
            assert sel.size == 0 or (sel.min() >= lo and sel.max() < hi)
        assert [gr.shard(100, r, ws) for r in range(ws)][-1][1] == 100
