"""Whole-program checking through the C ABI (include/mckg.h: mck_run_source).

The mirror of the reference driver path (/root/reference/proj/src/driver.cpp:87-161,
Machine::run machine.cpp:1180-1227): compile a CUDA-C program, interpret the
host thread on the CPU, run every grid on the B200 engine (K1 + fused race
detector + barrier-deadlock scan), and return the RunResult.  There is no CPU
execution path for device code: a launch without a CUDA device is reported in
``engine_error``.
"""
import ctypes
import json

from . import _abi


class RunOpts(ctypes.Structure):
    _fields_ = [
        ("step_limit", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("race_check", ctypes.c_int32),
        ("round_robin", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("max_threads_per_block", ctypes.c_int32),
        ("n_devices", ctypes.c_int32),
        ("devices", ctypes.c_int32 * 8),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("comm_id", ctypes.c_uint8 * 128),
        ("allgather", ctypes.c_void_p),
        ("allgather_ctx", ctypes.c_void_p),
        ("trace", ctypes.c_int32),
    ]


ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p)


def _lib():
    lib = _abi.load()
    if not getattr(lib, "_mck_bound", False):
        lib.mck_run_source.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(RunOpts),
                                       ctypes.POINTER(ctypes.c_void_p)]
        lib.mck_disassemble.argtypes = [ctypes.c_char_p, ctypes.c_char_p,
                                        ctypes.POINTER(ctypes.c_void_p)]
        lib.mck_free.argtypes = [ctypes.c_void_p]
        lib.mckg_comm_id.argtypes = [ctypes.c_void_p]
        lib._mck_bound = True
    return lib


def comm_id():
    """A fresh 128-byte NCCL communicator id (rank 0 makes it and broadcasts it)."""
    lib = _lib()
    buf = (ctypes.c_uint8 * 128)()
    _abi.check(lib.mckg_comm_id(buf), "mckg_comm_id")
    return bytes(buf)


def torch_allgather(group=None):
    """Host transport over torch.distributed (gloo): the `allgather` argument
    of run_source for ranks that share a GPU."""
    import torch
    import torch.distributed as dist

    def gather(send):
        world = dist.get_world_size(group)
        t = torch.frombuffer(bytearray(send), dtype=torch.uint8) if send else torch.empty(0, dtype=torch.uint8)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t, group=group)
        return b"".join(o.numpy().tobytes() for o in outs)
    return gather


def run_source(src, filename="test.cu", step_limit=0, race_check=True, device=0,
               round_robin=True, seed=0, devices=None, rank=0, world=1, comm=None, allgather=None,
               trace=False):
    """Machine::run on a source program -> dict (keys: see include/mckg.h).

    devices: list of CUDA ordinals to split every grid over (a repeated
    ordinal makes virtual devices on one GPU).
    rank/world: one process per GPU; this rank runs its block range of every
    grid and the ranks combine memory and reports over NCCL (comm = the id
    from comm_id() on rank 0) or over `allgather(bytes) -> bytes` (host
    transport, e.g. torch_allgather())."""
    lib = _lib()
    devs = list(devices or [])
    arr = (ctypes.c_int32 * 8)(*(devs + [0] * (8 - len(devs))))
    cid = (ctypes.c_uint8 * 128)(*(comm or bytes(128)))
    cb = None
    if allgather is not None:
        def _cb(ctx, send, n, recv):
            try:
                got = allgather(ctypes.string_at(send, n) if n else b"")
                ctypes.memmove(recv, got, len(got))
                return 0
            except Exception:  # noqa: BLE001 -- reported as an engine error by the library
                return 1
        cb = ALLGATHER(_cb)
    o = RunOpts(step_limit, seed, 1 if race_check else 0, 1 if round_robin else 0, device, 0, len(devs), arr,
                rank, world, cid, ctypes.cast(cb, ctypes.c_void_p) if cb else None, None, 1 if trace else 0)
    out = ctypes.c_void_p()
    rc = lib.mck_run_source(src.encode(), filename.encode(), ctypes.byref(o), ctypes.byref(out))
    _abi.check(rc, "mck_run_source")
    s = ctypes.string_at(out.value).decode()
    lib.mck_free(out)
    return json.loads(s)


def disassemble(src, filename="test.cu"):
    lib = _lib()
    out = ctypes.c_void_p()
    lib.mck_disassemble(src.encode(), filename.encode(), ctypes.byref(out))
    s = ctypes.string_at(out.value).decode()
    lib.mck_free(out)
    return s
