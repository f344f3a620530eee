"""K4 (mckg_scan_stuck) parity against the deadlock.cpp restatement."""
import numpy as np
import pytest

import oracle_bind as ob

pytestmark = pytest.mark.gpu


def _run(arr, nb, bd, bid_base=0):
    import torch
    from paper_1211_6193_b200 import race
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint32).reshape(-1).view(np.int32)).cuda()
    st = race.scan_stuck(t, nb, bd, bid_base)
    wm, dl = ob.port_scan_stuck(arr.reshape(-1), nb, bd, bid_base)
    assert np.array_equal(st.waiting_mask.reshape(-1), wm)
    assert np.array_equal(st.deadlocked, dl)
    return st


@pytest.mark.parametrize("bd", [1, 7, 32, 33, 100, 256, 1024])
def test_random_counts(bd):
    rng = np.random.default_rng(bd)
    nb = 37
    arr = rng.integers(3, 5, size=(nb, bd)).astype(np.uint32)
    arr[rng.random(nb) < 0.4] = 4  # uniform blocks: no deadlock
    _run(arr, nb, bd, bid_base=11)


def test_c4_pattern_closed_form():
    # if (v % 2) __syncthreads();  -> arrivals = v % 2 ; waiting = odd-v threads
    rng = np.random.default_rng(0)
    nb, bd = 512, 1024
    pat = rng.integers(0, 3, size=nb)
    v = rng.integers(0, 1 << 20, size=(nb, bd))
    v[pat == 0] &= ~1
    v[pat == 1] |= 1
    arr = (v % 2).astype(np.uint32)
    st = _run(arr, nb, bd)
    assert set(st.deadlocked.tolist()) == set(np.nonzero(pat == 2)[0].tolist()) - {
        b for b in np.nonzero(pat == 2)[0] if arr[b].min() == arr[b].max()}
