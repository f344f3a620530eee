"""Full-size C3 parity: the GPU detector's result on the whole 2^30-event trace
against the reference replay (TEST INFRASTRUCTURE ONLY -- imported by tests/
and by bench.py's cpu_baseline leg, never by the product).

The reference (oracle/_ref/libmckref.so: Machine::recordAccess/clearEpoch,
racecheck.cpp:9-73, unmodified) replays the trace chunk by chunk of blocks on
all host threads.  Shared objects are per block (device.cpp:33-38), so a
chunk's reported triples are exactly the slice of the whole run's set whose
object ids fall in the chunk, and the per-line first-detection timestamps of
the whole run are the MIN over the chunks.  Every chunk is compared with the
GPU's sorted triples slice; the merged line table is compared at the end.
"""
import time

import numpy as np

import oracle_bind as ob


def replay_full(gpu_triples, gpu_line_first, n_blocks, nthreads, chunk_blocks=1 << 16,
                max_blocks=None, obj_base=1, prefer_ref=True):
    """gpu_triples: TRIPLE_DTYPE array in std::set order (the whole run);
    gpu_line_first: uint64[65536].  Replays blocks [0, max_blocks or n_blocks)
    and returns a dict with the parity verdict and the replay's own timing
    (generation excluded)."""
    use_ref = prefer_ref and ob.ref() is not None
    fn = ob.ref_detect if use_ref else ob.port_detect
    todo = n_blocks if max_blocks is None else min(n_blocks, max_blocks)
    objs = gpu_triples["obj"]
    lf = np.full(ob.MAX_LINES, ob.TS_NONE, dtype=np.uint64)
    replay_s = 0.0
    n_ref = 0
    mismatch = None
    b = 0
    while b < todo:
        nb = min(chunk_blocks, todo - b)
        ev, bs = ob.gen_c3(b, nb)
        tr = ob.make_trace(ev, bs, ob.C3_SHMEM, obj_base=obj_base + b, bid_base=b)
        t0 = time.perf_counter()
        rc, tri, n, clf = fn(tr, nthreads=nthreads, capacity=nb * ob.C3_EVENTS_PER_BLOCK // 4 + 16)
        replay_s += time.perf_counter() - t0
        if rc != 0:
            mismatch = mismatch or f"replay rc={rc} at blocks {b}..{b + nb - 1}"
            break
        n_ref += n
        lo = np.searchsorted(objs, obj_base + b, side="left")
        hi = np.searchsorted(objs, obj_base + b + nb, side="left")
        got = gpu_triples[lo:hi]
        want = ob.sorted_triples(tri)
        if mismatch is None and (len(got) != len(want) or not np.array_equal(got, want)):
            mismatch = f"triples differ in blocks {b}..{b + nb - 1}: gpu {len(got)} vs reference {len(want)}"
        np.minimum(lf, clf, out=lf)
        b += nb
        del ev, bs, tr, tri
    full = todo == n_blocks
    lf_ok = bool(np.array_equal(lf, gpu_line_first)) if full else None
    if full and mismatch is None and len(gpu_triples) != n_ref:
        mismatch = f"triple count: gpu {len(gpu_triples)} vs reference {n_ref}"
    return {
        "checked_blocks": todo, "of_blocks": n_blocks, "events": todo * ob.C3_EVENTS_PER_BLOCK,
        "reference_triples": int(n_ref), "triples_equal": mismatch is None,
        "line_first_equal": lf_ok, "mismatch": mismatch,
        "kind": "reference" if use_ref else "port", "threads": nthreads, "replay_s": replay_s,
    }
