"""ctypes bindings to the CPU oracle (TEST INFRASTRUCTURE ONLY).

* ``liboracle.so``   -- the C restatement in oracle/ (detector.c, deadlock.c,
  tracegen.c); always built by ``__graft_entry__.build()``.
* ``_ref/libmckref.so`` -- the unmodified reference library (built from
  /root/reference by oracle/Makefile) behind oracle/ref_shim.cpp; present only
  where it could be built (travels to the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.
"""
import ctypes
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")

ACCESS_DTYPE = np.dtype([("w0", "<u4"), ("w1", "<u4"), ("line", "<i4"), ("sweep", "<u4")])
TRIPLE_DTYPE = np.dtype([("obj", "<u4"), ("byte", "<u4"), ("line", "<i4")])
MAX_LINES = 65536
TS_NONE = np.uint64(0xFFFFFFFFFFFFFFFF)
C3_EVENTS_PER_BLOCK = 1024
C3_SHMEM = 4096
C3_SEED = 0x12116193


class Trace(ctypes.Structure):
    _fields_ = [
        ("events", ctypes.c_void_p),
        ("block_start", ctypes.c_void_p),
        ("n_events", ctypes.c_uint64),
        ("n_blocks", ctypes.c_uint32),
        ("max_block_events", ctypes.c_uint32),
        ("obj_base", ctypes.c_uint32),
        ("bid_base", ctypes.c_uint32),
        ("shmem_bytes", ctypes.c_uint32),
        ("gid", ctypes.c_uint32),
    ]


def make_access(off, length, write, tid, epoch, line, sweep):
    w0 = (off & 0xFFFFF) | ((length & 0xF) << 20) | ((1 if write else 0) << 24)
    w1 = (tid & 0x7FF) | (epoch << 11)
    return (w0, w1, line, sweep)


def ts_key(sweep, bid, tid):
    return (int(sweep) << 32) | ((int(bid) & ((1 << 21) - 1)) << 11) | (int(tid) & 0x7FF)


def _lib(path):
    return ctypes.CDLL(path) if os.path.exists(path) else None


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        _port = _lib(os.path.join(ORACLE_DIR, "liboracle.so"))
        if _port is None:
            raise RuntimeError("oracle/liboracle.so missing: run __graft_entry__.build()")
        _port.oracle_detect_shared.argtypes = [ctypes.POINTER(Trace), ctypes.c_void_p,
                                               ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                               ctypes.c_void_p, ctypes.c_int]
        _port.oracle_scan_stuck.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.POINTER(ctypes.c_uint32)]
        _port.oracle_gen_c3.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_uint64]
        _port.oracle_gen_c5.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_uint64]
        _port.oracle_detect_global.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                               ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                               ctypes.c_void_p]
    return _port


def ref():
    """The reference library, or None where it was not built."""
    global _ref
    if _ref is None:
        _ref = _lib(os.path.join(ORACLE_DIR, "_ref", "libmckref.so"))
        if _ref is not None:
            _ref.mckref_replay_shared.argtypes = [ctypes.POINTER(Trace), ctypes.c_void_p,
                                                  ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                                  ctypes.c_void_p, ctypes.c_int]
            _ref.mckref_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                        ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
            _ref.mckref_free.argtypes = [ctypes.c_void_p]
    return _ref


def gen_c3(blk0, n_blocks, seed=C3_SEED):
    ev = np.zeros(n_blocks * C3_EVENTS_PER_BLOCK, dtype=ACCESS_DTYPE)
    bs = np.zeros(n_blocks + 1, dtype=np.uint64)
    port().oracle_gen_c3(ev.ctypes.data, bs.ctypes.data, blk0, n_blocks, seed)
    return ev, bs


GACCESS_DTYPE = np.dtype([("a", "<u8"), ("sweep", "<u4"), ("b", "<u4")])
GRACE_DTYPE = np.dtype([("addr", "<u8"), ("line", "<i4"), ("pad", "<i4")])
C5_EVENTS_PER_BLOCK = 4096


def make_gaccess(addr, length, write, tid, bid, line, sweep):
    a = ((addr & 0xFFFFFFFFFF) | ((length & 0xF) << 40) | ((1 if write else 0) << 44)
         | ((tid & 0x7FF) << 45) | ((line & 0xFF) << 56))
    return (a, sweep, (bid & 0xFFFFFF) | (((line >> 8) & 0xFF) << 24))


def gen_c5(blk0, n_blocks, n_total, seed=C3_SEED):
    ev = np.zeros(n_blocks * C5_EVENTS_PER_BLOCK, dtype=GACCESS_DTYPE)
    port().oracle_gen_c5(ev.ctypes.data, blk0, n_blocks, n_total, seed)
    return ev


def port_detect_global(ev, capacity=None):
    ev = np.ascontiguousarray(ev, dtype=GACCESS_DTYPE)
    if capacity is None:
        capacity = 4 * len(ev) + 16
    races = np.zeros(capacity, dtype=GRACE_DTYPE)
    n = ctypes.c_uint64(0)
    lf = np.full(MAX_LINES, TS_NONE, dtype=np.uint64)
    rc = port().oracle_detect_global(ev.ctypes.data, len(ev), races.ctypes.data, capacity, ctypes.byref(n),
                                     lf.ctypes.data)
    return rc, races[: min(n.value, capacity)], n.value, lf


def make_trace(events, block_start, shmem_bytes, obj_base=1, bid_base=0, gid=1):
    counts = np.diff(block_start.astype(np.int64)) if len(block_start) > 1 else np.zeros(0)
    t = Trace(events.ctypes.data, block_start.ctypes.data, len(events), len(block_start) - 1,
              int(counts.max()) if len(counts) else 0, obj_base, bid_base, shmem_bytes, gid)
    t._keep = (events, block_start)
    return t


def _detect(fn, trace, nthreads, capacity):
    if capacity is None:
        capacity = max(16, 8 * int(trace.n_events) + 16)
    tri = np.zeros(capacity, dtype=TRIPLE_DTYPE)
    n = ctypes.c_uint64(0)
    lf = np.full(MAX_LINES, TS_NONE, dtype=np.uint64)
    rc = fn(ctypes.byref(trace), tri.ctypes.data, capacity, ctypes.byref(n), lf.ctypes.data, nthreads)
    return rc, tri[: min(n.value, capacity)], n.value, lf


def port_detect(trace, nthreads=1, capacity=None):
    return _detect(port().oracle_detect_shared, trace, nthreads, capacity)


def ref_detect(trace, nthreads=1, capacity=None):
    return _detect(ref().mckref_replay_shared, trace, nthreads, capacity)


def port_scan_stuck(arrivals, n_blocks, block_dim, bid_base=0):
    words = (block_dim + 31) // 32
    wm = np.zeros(n_blocks * words, dtype=np.uint32)
    dl = np.zeros(max(1, n_blocks), dtype=np.uint32)
    n = ctypes.c_uint32(0)
    a = np.ascontiguousarray(arrivals, dtype=np.uint32)
    rc = port().oracle_scan_stuck(a.ctypes.data, n_blocks, block_dim, bid_base, wm.ctypes.data,
                                  dl.ctypes.data, ctypes.byref(n))
    assert rc == 0
    return wm, dl[: n.value]


def ref_run(src, filename="test.cu", policy="rr", seed=0, step_limit=50_000_000, race_check=True,
            capture=True, trace=False):
    """Machine::run of the reference on a source program -> dict (see ref_shim.cpp)."""
    lib = ref()
    out = ctypes.c_void_p()
    lib.mckref_run(src.encode(), filename.encode(), 1 if policy == "rr" else 0, seed, step_limit,
                   1 if race_check else 0, (1 if capture else 0) | (2 if trace else 0), ctypes.byref(out))
    s = ctypes.string_at(out.value).decode()
    lib.mckref_free(out)
    return json.loads(s)


def sorted_triples(tri):
    """std::set<tuple<ObjectId,int64_t,int>> order (machine.hpp:91)."""
    if len(tri) == 0:
        return np.zeros(0, dtype=TRIPLE_DTYPE)
    order = np.lexsort((tri["line"], tri["byte"], tri["obj"]))
    return tri[order]


def race_lines(line_first):
    """Race diagnostic lines in report order (first detection)."""
    idx = np.nonzero(line_first != TS_NONE)[0]
    return [int(l) for l in idx[np.argsort(line_first[idx], kind="stable")]]


def trace_from_run(run, gid=None):
    """Group the shared events a reference run captured into per-grid traces.

    Returns {gid: (events, block_start, obj_base, n_blocks)}; blocks of a grid
    own consecutive objects (device.cpp:33-38)."""
    out = {}
    evs = run["events"]
    grids = sorted({e[0] for e in evs}) if gid is None else [gid]
    for g in grids:
        ge = [e for e in evs if e[0] == g]
        if not ge:
            continue
        nb = max(e[1] for e in ge) + 1
        objs = {}
        for e in ge:
            objs[e[1]] = e[3]
        base = min(objs[b] - b for b in objs)
        rows = sorted(ge, key=lambda e: (e[1], e[10]))  # block-major, step order
        arr = np.zeros(len(rows), dtype=ACCESS_DTYPE)
        counts = np.zeros(nb, dtype=np.int64)
        for i, e in enumerate(rows):
            arr[i] = make_access(e[4], e[5], e[6], e[2], e[7], e[8], e[9])
            counts[e[1]] += 1
        bs = np.zeros(nb + 1, dtype=np.uint64)
        bs[1:] = np.cumsum(counts)
        out[g] = (arr, bs, base, nb)
    return out
