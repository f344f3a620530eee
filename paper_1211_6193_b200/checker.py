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

import numpy as np

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
        ("global_race_check", ctypes.c_int32),
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


def _opts(step_limit=0, race_check=True, device=0, round_robin=True, seed=0, devices=None, rank=0,
          world=1, comm=None, allgather=None, trace=False, global_race_check=False):
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
                rank, world, cid, ctypes.cast(cb, ctypes.c_void_p) if cb else None, None, 1 if trace else 0,
                1 if global_race_check else 0)
    o._keep = cb
    return o


def run_source(src, filename="test.cu", **kw):
    """Machine::run on a source program -> dict (keys: see include/mckg.h).

    Keyword options (RunOptions): step_limit, race_check, device,
    round_robin, seed, trace; devices: list of CUDA ordinals to split every
    grid over (a repeated ordinal makes virtual devices on one GPU);
    rank/world: one process per GPU; this rank runs its block range of every
    grid and the ranks combine memory and reports over NCCL (comm = the id
    from comm_id() on rank 0) or over `allgather(bytes) -> bytes` (host
    transport, e.g. torch_allgather())."""
    lib = _lib()
    o = _opts(**kw)
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


# ---- result records (mck_run / mck_result_*: no JSON) ----
TRIPLE_DTYPE = np.dtype([("obj", "<u4"), ("byte", "<u4"), ("line", "<i4")])
CATEGORIES = ("race", "deadlock", "memBoundary", "undefinedBehavior", "apiError")
STUCK_KINDS = ("barrier", "host", "stream")


class Summary(ctypes.Structure):
    _fields_ = [("exit_code", ctypes.c_int32), ("stuck", ctypes.c_int32), ("has_main_return", ctypes.c_int32),
                ("frontend_line", ctypes.c_int32), ("main_return", ctypes.c_int64), ("steps", ctypes.c_uint64),
                ("n_diags", ctypes.c_uint64), ("n_stuck", ctypes.c_uint64), ("n_reported", ctypes.c_uint64),
                ("n_trace", ctypes.c_uint64), ("output_bytes", ctypes.c_uint64), ("output", ctypes.c_char_p),
                ("engine_error", ctypes.c_char_p), ("frontend_stage", ctypes.c_char_p),
                ("frontend_message", ctypes.c_char_p), ("report_text", ctypes.c_char_p),
                ("engine_note", ctypes.c_char_p)]


class DiagRec(ctypes.Structure):
    _fields_ = [("category", ctypes.c_int32), ("severity", ctypes.c_int32), ("line", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("sweep", ctypes.c_uint64), ("message", ctypes.c_char_p)]


class StuckRec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gid", ctypes.c_uint32), ("bid", ctypes.c_int32), ("sid", ctypes.c_uint32),
                ("n_waiting", ctypes.c_uint64), ("n_missing", ctypes.c_uint64),
                ("waiting", ctypes.POINTER(ctypes.c_int32)), ("missing", ctypes.POINTER(ctypes.c_int32)),
                ("reason", ctypes.c_char_p), ("item", ctypes.c_char_p)]


def _rec_lib():
    lib = _lib()
    if not getattr(lib, "_mck_rec_bound", False):
        vp = ctypes.c_void_p
        lib.mck_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(RunOpts), ctypes.POINTER(vp)]
        lib.mck_result_summary.argtypes = [vp, ctypes.POINTER(Summary)]
        lib.mck_result_diag.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(DiagRec)]
        lib.mck_result_stuck.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(StuckRec)]
        lib.mck_result_reported.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, vp]
        lib.mck_result_trace.argtypes = [vp, ctypes.c_uint64]
        lib.mck_result_trace.restype = ctypes.c_char_p
        lib.mck_result_stats.argtypes = [vp, ctypes.POINTER(RunStats)]
        lib.mck_result_free.argtypes = [vp]
        lib.mck_result_free.restype = None
        lib._mck_rec_bound = True
    return lib


class RunStats(ctypes.Structure):
    _fields_ = [("host_steps", ctypes.c_uint64), ("device_steps", ctypes.c_uint64),
                ("barrier_rules", ctypes.c_uint64), ("dispatches", ctypes.c_uint64),
                ("shared_events", ctypes.c_uint64), ("grids", ctypes.c_uint64), ("sweeps", ctypes.c_uint64),
                ("grid_ms", ctypes.c_double), ("kernel_launches", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("block_sweeps", ctypes.c_uint64), ("solo_sweeps", ctypes.c_uint64),
                ("block_cycles", ctypes.c_uint64), ("solo_cycles", ctypes.c_uint64)]


def run(src, filename="test.cu", stuck_lists=None, **kw):
    """Machine::run through the result-record ABI.  Same keys as run_source
    (exit, output, steps, stuck, main_return, diags, stuck_reports,
    report_text, engine_error, trace, stats), but `reported` is a numpy
    array of (obj, byte, line) records in std::set order -- fit for millions
    of triples.  stuck_lists=N: waiting/missing lists for the first N stuck
    reports only (every report keeps kind, gid and bid)."""
    lib = _rec_lib()
    o = _opts(**kw)
    h = ctypes.c_void_p()
    _abi.check(lib.mck_run(src.encode(), filename.encode(), ctypes.byref(o), ctypes.byref(h)), "mck_run")
    try:
        sm = Summary()
        _abi.check(lib.mck_result_summary(h, ctypes.byref(sm)), "mck_result_summary")
        if sm.frontend_stage:
            return {"frontend_error": f"{sm.frontend_stage.decode()}: {sm.frontend_message.decode()}",
                    "line": sm.frontend_line, "exit": sm.exit_code}
        diags = []
        for i in range(sm.n_diags):
            d = DiagRec()
            _abi.check(lib.mck_result_diag(h, i, ctypes.byref(d)), "mck_result_diag")
            diags.append({"cat": CATEGORIES[d.category], "sev": "error" if d.severity == 0 else "warning",
                          "msg": d.message.decode(), "line": d.line})
        stuck = []
        for i in range(sm.n_stuck):
            r = StuckRec()
            _abi.check(lib.mck_result_stuck(h, i, ctypes.byref(r)), "mck_result_stuck")
            full = stuck_lists is None or i < stuck_lists
            stuck.append({"kind": STUCK_KINDS[r.kind], "gid": r.gid, "bid": r.bid,
                          "waiting": [r.waiting[k] for k in range(r.n_waiting)] if full else None,
                          "missing": [r.missing[k] for k in range(r.n_missing)] if full else None,
                          "n_waiting": r.n_waiting, "n_missing": r.n_missing, "reason": r.reason.decode()})
        st = RunStats()
        _abi.check(lib.mck_result_stats(h, ctypes.byref(st)), "mck_result_stats")
        stats = {f: getattr(st, f) for f, _ in RunStats._fields_ if f != "pad"}
        rep = np.zeros(sm.n_reported, dtype=TRIPLE_DTYPE)
        if sm.n_reported:
            _abi.check(lib.mck_result_reported(h, 0, sm.n_reported, rep.ctypes.data), "mck_result_reported")
        return {"exit": sm.exit_code, "output": ctypes.string_at(sm.output, sm.output_bytes).decode(),
                "steps": sm.steps, "stuck": bool(sm.stuck),
                "main_return": sm.main_return if sm.has_main_return else None,
                "engine_error": sm.engine_error.decode(), "engine_note": sm.engine_note.decode(),
                "diags": diags, "stuck_reports": stuck,
                "report_text": sm.report_text.decode(), "reported": rep,
                "trace": [lib.mck_result_trace(h, i).decode() for i in range(sm.n_trace)], "stats": stats}
    finally:
        lib.mck_result_free(h)


class OracleResult(ctypes.Structure):
    _fields_ = [("oracle_race", ctypes.c_int32), ("detector_race", ctypes.c_int32), ("aborted", ctypes.c_int32),
                ("frontend_error", ctypes.c_int32), ("interleavings", ctypes.c_uint64), ("error", ctypes.c_char * 256)]


def oracle_race(src, filename="test.cu", max_interleavings=1_000_000, max_threads=3, max_accesses_per_thread=8):
    """oracleRace (oracle.hpp:34) through mck_oracle: every interleaving of the
    grid's shared accesses, explored on the GPU."""
    lib = _lib()
    lib.mck_oracle.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32,
                               ctypes.POINTER(OracleResult)]
    r = OracleResult()
    _abi.check(lib.mck_oracle(src.encode(), filename.encode(), max_interleavings, max_threads,
                              max_accesses_per_thread, ctypes.byref(r)), "mck_oracle")
    if r.frontend_error:
        return {"frontend_error": r.error.decode()}
    return {"oracle_race": bool(r.oracle_race), "detector_race": bool(r.detector_race),
            "interleavings": int(r.interleavings), "aborted": bool(r.aborted), "error": r.error.decode()}
