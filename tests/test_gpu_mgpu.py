"""The multi-GPU C-ABI entry points (mckg_comm_init, mckg_detect_shared_mgpu,
mckg_detect_global_mgpu) on a one-rank NCCL communicator: the library-owned
exchange must leave the single-GPU results unchanged.  (Two ranks need two
GPUs; the multi-rank dataflow is covered by tests/test_gpu_multirank.py over
gloo and tests/test_dist_exchange.py.)"""
import numpy as np
import pytest

import oracle_bind as ob

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    import torch
    from paper_1211_6193_b200 import checker, race
    torch.cuda.set_device(0)
    c = race.Comm(checker.comm_id(), 0, 1, 0)
    yield c
    c.close()


def test_shared_mgpu_equals_single(comm):
    from paper_1211_6193_b200 import race
    ev, bs = race.gen_c3(0, 2048)
    tr = race.make_trace(ev, bs, ob.C3_SHMEM, max_block_events=1024)
    a = race.fetch(race.detect_shared_async(tr, race.RaceOut(1 << 20)))
    b = race.fetch(race.detect_shared_mgpu(comm, tr, race.RaceOut(1 << 20)))
    assert a.n_triples > 0 and a.n_triples == b.n_triples
    assert np.array_equal(a.triples, b.triples) and np.array_equal(a.line_first, b.line_first)


def test_global_mgpu_equals_single(comm):
    from paper_1211_6193_b200 import global_race as gr
    ev = gr.gen_c5(0, 256, 256)
    space = 256 * 65536
    r1 = gr.fetch(gr.detect(ev, 0, gr.GlobalOut(1 << 20).reset()))
    r2 = gr.fetch(gr.detect_mgpu(comm, ev, space, gr.GlobalOut(1 << 20).reset()))
    o1 = np.lexsort((r1[0]["line"], r1[0]["addr"]))
    o2 = np.lexsort((r2[0]["line"], r2[0]["addr"]))
    assert r1[1] > 0 and r1[1] == r2[1] and r2[3] == 0
    assert np.array_equal(r1[0][o1], r2[0][o2]) and np.array_equal(r1[2], r2[2])
