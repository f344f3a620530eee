"""Cross-block global-memory race detection across ranks (BASELINE config 5,
SURVEY §8(e) / Appendix E; an extension: the reference checks shared memory
only, so parity is unpinned and the checker is oracle/global_detector.c).

Pipeline per rank (one process per GPU, torch.distributed for the plumbing):
  1. records of this rank's shard of simulated blocks (mckg_gen_c5 or a trace);
  2. K3 mckg_partition_global: bucket by owner rank (address-range partition);
  3. count exchange + all_to_all_single of the 16-byte records (NCCL over
     NVLink on GPUs; gloo in the CPU tests);
  4. K6 mckg_detect_global on the received records (sort by word + run scan);
  5. the per-line first-detection table is MIN-all-reduced; the reported
     (byte, line) sets are disjoint across ranks (each byte has one owner).
"""
import ctypes

import numpy as np
import torch

from . import _abi

GACCESS_DTYPE = np.dtype([("a", "<u8"), ("sweep", "<u4"), ("b", "<u4")])
GRACE_DTYPE = np.dtype([("addr", "<u8"), ("line", "<i4"), ("pad", "<i4")])
ADDR_SPACE_C5 = 1 << 36  # 64 GiB


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _s(stream):
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def owner_of(addr, n_ranks, space):
    """Address-range owner (same formula as K3)."""
    return np.minimum((addr.astype(np.uint64) * np.uint64(n_ranks)) // np.uint64(space), n_ranks - 1)


def addr_range(rank, n_ranks, space):
    """[lo, hi) of the addresses rank owns: owner(a) == rank  <=>  a*P // A == rank."""
    lo = -(-rank * space // n_ranks)
    hi = -(-(rank + 1) * space // n_ranks)
    return lo, hi


def gen_c5(blk0, n_blocks, n_total, seed=0x12116193, device="cuda", stream=None):
    ev = torch.empty((n_blocks * _abi.C5_EVENTS_PER_BLOCK, 4), dtype=torch.int32, device=device)
    _abi.check(_abi.load().mckg_gen_c5(_p(ev), blk0, n_blocks, n_total, seed, _s(stream)), "mckg_gen_c5")
    return ev


def partition(ev, n_ranks, space, stream=None):
    """K3: records grouped by owner rank + per-rank counts (device tensors)."""
    out = torch.empty_like(ev)
    counts = torch.zeros(max(1, n_ranks), dtype=torch.int64, device=ev.device)
    _abi.check(_abi.load().mckg_partition_global(_p(ev), ev.shape[0], n_ranks, space, _p(out), _p(counts),
                                                 _s(stream)), "mckg_partition_global")
    return out, counts


def exchange(grouped, counts, group=None):
    """Count exchange, then all_to_all_single of the grouped 16-byte records.

    `grouped` is [n, 4] int32 (records grouped by destination rank),
    `counts` the per-destination sizes.  Works on CUDA tensors (NCCL) and CPU
    tensors (gloo)."""
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    # gloo (CPU tests, one-GPU dry runs) moves host tensors; NCCL moves HBM
    host = dist.get_backend(group) == "gloo"
    dev = grouped.device
    send = counts.to(torch.int64)
    if host:
        send = send.cpu()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    s_list = [int(x) for x in send.cpu().tolist()]
    r_list = [int(x) for x in recv.cpu().tolist()]
    src = grouped.contiguous().cpu() if host else grouped.contiguous()
    out = torch.empty((sum(r_list), 4), dtype=grouped.dtype, device=src.device)
    assert len(s_list) == ws
    dist.all_to_all_single(out, src, r_list, s_list, group=group)
    return out.to(dev) if host else out


class GlobalOut:
    def __init__(self, capacity, device="cuda"):
        self.capacity = int(capacity)
        self.races = torch.empty((max(1, self.capacity), 4), dtype=torch.int32, device=device)
        self.n = torch.zeros(1, dtype=torch.int64, device=device)
        self.line_first = torch.full((_abi.MAX_LINES,), -1, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)

    def reset(self):
        self.line_first.fill_(-1)
        self.status.zero_()
        return self


def detect(ev, addr_lo, out, stream=None):
    """K6 on one rank's records (device)."""
    _abi.check(_abi.load().mckg_detect_global(_p(ev), ev.shape[0], addr_lo, _p(out.races), out.capacity,
                                              _p(out.n), _p(out.line_first), _p(out.status), _s(stream)),
               "mckg_detect_global")
    return out


def detect_mgpu(comm, ev, addr_space, out, stream=None):
    """mckg_detect_global_mgpu: owner partition, all-to-all over NCCL, K6 on
    the owned range and the line-table MIN, all inside the library."""
    _abi.check(_abi.load().mckg_detect_global_mgpu(comm.handle, _p(ev), ev.shape[0], addr_space, _p(out.races),
                                                   out.capacity, _p(out.n), _p(out.line_first), _p(out.status),
                                                   _s(stream)), "mckg_detect_global_mgpu")
    return out


def min_allreduce_u64(t, group=None):
    """MIN all-reduce of uint64 values stored in an int64 tensor."""
    import torch.distributed as dist
    t.bitwise_xor_(-(1 << 63))
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    t.bitwise_xor_(-(1 << 63))
    return t


def fetch(out):
    n = int(out.n.item())
    nc = min(n, out.capacity)
    races = out.races[:nc].cpu().numpy().view(GRACE_DTYPE).reshape(-1).copy()
    lf = out.line_first.cpu().numpy().view(np.uint64).copy()
    return races, n, lf, int(out.status.item())


def shard(n_blocks, rank, ws):
    """Contiguous block range of a rank (block b -> rank b * ws // n_blocks)."""
    return n_blocks * rank // ws, n_blocks * (rank + 1) // ws
