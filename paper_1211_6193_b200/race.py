"""Device-side race / deadlock checking through the C ABI (include/mckg.h).

torch supplies device memory and streams only; every computation runs in the
sm_100a kernels of libmckg.so.  Mirrors the reference's observable outputs:

* ``RaceState::reported`` (machine.hpp:91)      -> ``RaceResult.triples`` (sorted)
* Race diagnostics in first-detection order
  (addDiagnostic, machine.cpp:41-46)            -> ``RaceResult.race_lines``
* ``StuckReport`` BarrierDeadlock entries
  (deadlock.cpp:12-34)                          -> ``StuckResult``
"""
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi

TRIPLE_DTYPE = np.dtype([("obj", "<u4"), ("byte", "<u4"), ("line", "<i4")])


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream_handle(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class RaceOut:
    """Caller-owned device outputs of mckg_detect_shared."""

    def __init__(self, capacity, device="cuda"):
        self.capacity = int(capacity)
        self.triples = torch.empty((max(1, self.capacity), 3), dtype=torch.int32, device=device)
        self.n_triples = torch.zeros(1, dtype=torch.int64, device=device)
        self.line_first = torch.empty(_abi.MAX_LINES, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self._c = _abi.RaceOut(self.triples.data_ptr(), self.capacity, self.n_triples.data_ptr(),
                               self.line_first.data_ptr(), self.status.data_ptr())

    def reset(self, stream=None):
        _abi.check(_abi.load().mckg_race_out_reset(ctypes.byref(self._c), _stream_handle(stream)),
                   "mckg_race_out_reset")
        return self


@dataclass
class RaceResult:
    triples: np.ndarray      # TRIPLE_DTYPE, std::set order
    n_triples: int
    line_first: np.ndarray   # uint64 [65536], TS_NONE = never raced
    status: int

    @property
    def race_lines(self):
        lf = self.line_first
        idx = np.nonzero(lf != np.uint64(_abi.TS_NONE))[0]
        return [int(l) for l in idx[np.argsort(lf[idx], kind="stable")]]

    def diagnostics(self, filename):
        """The Race diagnostic messages, in the reference's order (racecheck.cpp:37-40)."""
        return [f"Possible race on shared device memory detected at {filename}:{l}."
                for l in self.race_lines]


def make_trace(events, block_start, shmem_bytes, obj_base=1, bid_base=0, gid=1,
               max_block_events=None):
    """Build an mckg_trace over device tensors.

    events: int32 tensor [n, 4] (the 16-byte mckg_access records) on cuda.
    block_start: int64 tensor [n_blocks + 1] on cuda."""
    assert events.is_cuda and block_start.is_cuda
    assert events.dtype == torch.int32 and events.dim() == 2 and events.shape[1] == 4
    assert block_start.dtype == torch.int64
    n_blocks = block_start.numel() - 1
    if max_block_events is None:
        max_block_events = int(torch.diff(block_start).max().item()) if n_blocks > 0 else 0
    t = _abi.Trace(events.data_ptr(), block_start.data_ptr(), events.shape[0], n_blocks,
                   int(max_block_events), obj_base, bid_base, shmem_bytes, gid)
    t._keep = (events, block_start)
    return t


def detect_shared_async(trace, out, stream=None, reset=True):
    """Launch K2 on `stream`; results stay on the device in `out`."""
    lib = _abi.load()
    if reset:
        out.reset(stream)
    _abi.check(lib.mckg_detect_shared(ctypes.byref(trace), ctypes.byref(out._c),
                                      _stream_handle(stream)), "mckg_detect_shared")
    return out


def fetch(out, obj_base=1, sort=True, stream=None):
    """Copy the device results to host (sorted into std::set order on device)."""
    n = int(out.n_triples.item())
    status = int(out.status.item())
    nc = min(n, out.capacity)
    if (sort or status & _abi.STATUS_DUP) and nc > 0:
        uniq = out.n_triples if status & _abi.STATUS_DUP else None
        _abi.check(_abi.load().mckg_sort_triples(_ptr(out.triples), nc, obj_base, _ptr(uniq),
                                                 _stream_handle(stream)), "mckg_sort_triples")
        if uniq is not None:
            n = nc = int(out.n_triples.item())
            status &= ~_abi.STATUS_DUP
    tri = out.triples[:nc].cpu().numpy().view(TRIPLE_DTYPE).reshape(-1)
    lf = out.line_first.cpu().numpy().view(np.uint64)
    return RaceResult(tri.copy(), n, lf.copy(), status)


def detect_shared(events, block_start, shmem_bytes, obj_base=1, bid_base=0, gid=1,
                  capacity=None, max_block_events=None):
    """Synchronous convenience wrapper: device trace in, host RaceResult out."""
    trace = make_trace(events, block_start, shmem_bytes, obj_base, bid_base, gid, max_block_events)
    if capacity is None:
        capacity = 8 * events.shape[0] + 16
    out = RaceOut(capacity, device=events.device)
    detect_shared_async(trace, out)
    return fetch(out, obj_base)


def detect_shared_host(events_np, block_start_np, shmem_bytes, obj_base=1, bid_base=0, gid=1,
                       capacity=None):
    """Host buffers in, host results out (mckg_detect_shared_host)."""
    lib = _abi.load()
    ev = np.ascontiguousarray(events_np)
    bs = np.ascontiguousarray(block_start_np, dtype=np.uint64)
    n_blocks = len(bs) - 1
    mbe = int(np.diff(bs.astype(np.int64)).max()) if n_blocks > 0 else 0
    t = _abi.Trace(ev.ctypes.data, bs.ctypes.data, len(ev), n_blocks, mbe, obj_base, bid_base,
                   shmem_bytes, gid)
    if capacity is None:
        capacity = 8 * len(ev) + 16
    tri = np.zeros(capacity, dtype=TRIPLE_DTYPE)
    n = ctypes.c_uint64(0)
    lf = np.zeros(_abi.MAX_LINES, dtype=np.uint64)
    st = ctypes.c_uint32(0)
    _abi.check(lib.mckg_detect_shared_host(ctypes.byref(t), tri.ctypes.data, capacity,
                                           ctypes.byref(n), lf.ctypes.data, ctypes.byref(st)),
               "mckg_detect_shared_host")
    nc = min(n.value, capacity)
    tri = tri[:nc]
    order = np.lexsort((tri["line"], tri["byte"], tri["obj"]))
    return RaceResult(tri[order], n.value, lf, st.value)


@dataclass
class StuckResult:
    waiting_mask: np.ndarray  # uint32 [n_blocks, words]
    deadlocked: np.ndarray    # ascending bids

    def waiting_tids(self, b, block_dim):
        m = self.waiting_mask[b]
        return [t for t in range(block_dim) if (m[t // 32] >> (t % 32)) & 1]

    def missing_tids(self, b, block_dim):
        m = self.waiting_mask[b]
        return [t for t in range(block_dim) if not (m[t // 32] >> (t % 32)) & 1]


def scan_stuck_async(arrivals, n_blocks, block_dim, bid_base=0, stream=None):
    assert arrivals.is_cuda and arrivals.dtype == torch.int32
    words = (block_dim + 31) // 32
    wm = torch.empty((max(1, n_blocks), words), dtype=torch.int32, device=arrivals.device)
    dl = torch.empty(max(1, n_blocks), dtype=torch.int32, device=arrivals.device)
    ndl = torch.zeros(1, dtype=torch.int32, device=arrivals.device)
    _abi.check(_abi.load().mckg_scan_stuck(_ptr(arrivals), n_blocks, block_dim, bid_base, _ptr(wm),
                                           _ptr(dl), _ptr(ndl), _stream_handle(stream)),
               "mckg_scan_stuck")
    return wm, dl, ndl


def scan_stuck(arrivals, n_blocks, block_dim, bid_base=0):
    wm, dl, ndl = scan_stuck_async(arrivals, n_blocks, block_dim, bid_base)
    n = int(ndl.item())
    return StuckResult(wm[:n_blocks].cpu().numpy().view(np.uint32),
                       dl[:n].cpu().numpy().view(np.uint32).copy())


def gen_c3(blk0, n_blocks, seed=_abi.C3_SEED, device="cuda", stream=None):
    """Synthetic config-3 trace generated on the device."""
    ev = torch.empty((n_blocks * _abi.C3_EVENTS_PER_BLOCK, 4), dtype=torch.int32, device=device)
    bs = torch.empty(n_blocks + 1, dtype=torch.int64, device=device)
    _abi.check(_abi.load().mckg_gen_c3(_ptr(ev), _ptr(bs), blk0, n_blocks, seed,
                                       _stream_handle(stream)), "mckg_gen_c3")
    return ev, bs


class Comm:
    """The library-owned NCCL communicator of the multi-GPU entry points
    (mckg_comm_init): one process per GPU; `comm_id` is checker.comm_id() of
    rank 0, broadcast by the launcher."""

    def __init__(self, comm_id, rank, world, device):
        lib = _abi.load()
        buf = (ctypes.c_uint8 * 128)(*comm_id)
        self._h = ctypes.c_void_p()
        _abi.check(lib.mckg_comm_init(buf, rank, world, device, ctypes.byref(self._h)), "mckg_comm_init")
        self.rank, self.world, self.device = rank, world, device

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            _abi.load().mckg_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def detect_shared_mgpu(comm, trace, out, stream=None, reset=True):
    """mckg_detect_shared_mgpu: this rank's shard + the line-table MIN over ranks."""
    lib = _abi.load()
    if reset:
        out.reset(stream)
    _abi.check(lib.mckg_detect_shared_mgpu(comm.handle, ctypes.byref(trace), ctypes.byref(out._c),
                                           _stream_handle(stream)), "mckg_detect_shared_mgpu")
    return out
