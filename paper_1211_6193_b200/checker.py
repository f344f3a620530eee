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
    ]


def _lib():
    lib = _abi.load()
    if not getattr(lib, "_mck_bound", False):
        lib.mck_run_source.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(RunOpts),
                                       ctypes.POINTER(ctypes.c_void_p)]
        lib.mck_disassemble.argtypes = [ctypes.c_char_p, ctypes.c_char_p,
                                        ctypes.POINTER(ctypes.c_void_p)]
        lib.mck_free.argtypes = [ctypes.c_void_p]
        lib._mck_bound = True
    return lib


def run_source(src, filename="test.cu", step_limit=0, race_check=True, device=0,
               round_robin=True, seed=0):
    """Machine::run on a source program -> dict (keys: see include/mckg.h)."""
    lib = _lib()
    o = RunOpts(step_limit, seed, 1 if race_check else 0, 1 if round_robin else 0, device, 0)
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
