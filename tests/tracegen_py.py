"""Random block-segmented access traces for parity tests (test infrastructure).

Each block's events are emitted in timestamp order (sweep increasing, epochs
non-decreasing), as the interpreter produces them."""
import numpy as np

import oracle_bind as ob


def random_trace(seed, n_blocks=8, threads=32, shmem=256, epochs=3, per_epoch=64,
                 kinds=("int", "char", "long", "short", "mis"), p_write=0.4, hot=0.3,
                 empty_blocks=0.0, sweep0=0):
    rng = np.random.default_rng(seed)
    rows = []
    counts = []
    sweep = sweep0
    for b in range(n_blocks):
        if rng.random() < empty_blocks:
            counts.append(0)
            continue
        n = 0
        for e in range(epochs):
            k = int(rng.integers(0, per_epoch + 1))
            # (sweep, tid) pairs strictly increasing
            tids = np.sort(rng.integers(0, threads, size=k))
            for tid in tids:
                kind = kinds[int(rng.integers(0, len(kinds)))]
                ln = {"int": 4, "char": 1, "long": 8, "short": 2, "mis": 4}[kind]
                if shmem < ln:
                    continue
                if rng.random() < hot:
                    off = int(rng.integers(0, min(shmem - ln + 1, 16)))
                else:
                    off = int(rng.integers(0, shmem - ln + 1))
                if kind != "mis" and kind != "char":
                    off -= off % ln
                w = rng.random() < p_write
                line = int(rng.integers(10, 30))
                sweep += int(rng.integers(0, 2))
                rows.append(ob.make_access(off, ln, w, int(tid), e, line, sweep))
                n += 1
            sweep += 3
        counts.append(n)
    ev = np.array(rows, dtype=ob.ACCESS_DTYPE) if rows else np.zeros(0, dtype=ob.ACCESS_DTYPE)
    bs = np.zeros(n_blocks + 1, dtype=np.uint64)
    bs[1:] = np.cumsum(counts)
    return ev, bs
