"""ctypes view of include/mckg.h (the C ABI of libmckg.so).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a)
into ``paper_1211_6193_b200/libmckg.so``.  There is no CPU fallback: if the
library is missing, importing the device entry points raises.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MCKG_LIB: an alternative build of the same library (kernel experiments)
LIB_PATH = os.environ.get("MCKG_LIB") or os.path.join(_HERE, "libmckg.so")

MCKG_OK = 0
MCKG_E_ARG = 1
MCKG_E_RANGE = 2
MCKG_E_CUDA = 3
MCKG_E_OVERFLOW = 4
MCKG_E_ORDER = 5
MAX_LINES = 65536
TS_NONE = 0xFFFFFFFFFFFFFFFF
C3_EVENTS_PER_BLOCK = 1024
C3_SHMEM = 4096
C3_SEED = 0x12116193
C5_EVENTS_PER_BLOCK = 4096
C5_RANGE = 65536

STATUS_OVERFLOW = 1
STATUS_RANGE = 2
STATUS_ORDER = 4
STATUS_DUP = 8

EXPORTS = [
    "mckg_abi_version",
    "mckg_last_error",
    "mckg_device_count",
    "mckg_get_launch_stats",
    "mckg_set_debug",
    "mckg_race_out_reset",
    "mckg_detect_shared",
    "mckg_detect_shared_host",
    "mckg_sort_triples",
    "mckg_scan_stuck",
    "mckg_gen_c3",
    "mckg_gen_c5",
    "mckg_partition_global",
    "mckg_detect_global",
    "mckg_comm_id",
    "mckg_comm_init",
    "mckg_comm_destroy",
    "mckg_detect_shared_mgpu",
    "mckg_detect_global_mgpu",
    "mck_run_source",
    "mck_disassemble",
    "mck_free",
    "mck_run",
    "mck_oracle",
    "mck_result_summary",
    "mck_result_diag",
    "mck_result_stuck",
    "mck_result_reported",
    "mck_result_stats",
    "mck_result_trace",
    "mck_result_free",
]


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


class RaceOut(ctypes.Structure):
    _fields_ = [
        ("triples", ctypes.c_void_p),
        ("capacity", ctypes.c_uint64),
        ("n_triples", ctypes.c_void_p),
        ("line_first", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


class LaunchStats(ctypes.Structure):
    _fields_ = [
        ("kernels", ctypes.c_uint32),
        ("grid", ctypes.c_uint32),
        ("block", ctypes.c_uint32),
        ("smem_bytes", ctypes.c_uint32),
    ]


class MckgError(RuntimeError):
    pass


_lib = None


def load():
    """Load libmckg.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MckgError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
    lib.mckg_abi_version.restype = ctypes.c_int
    lib.mckg_last_error.restype = ctypes.c_char_p
    lib.mckg_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.mckg_get_launch_stats.argtypes = [ctypes.POINTER(LaunchStats)]
    lib.mckg_race_out_reset.argtypes = [ctypes.POINTER(RaceOut), vp]
    lib.mckg_set_debug.argtypes = [u32]
    lib.mckg_set_debug.restype = None
    lib.mckg_detect_shared.argtypes = [ctypes.POINTER(Trace), ctypes.POINTER(RaceOut), vp]
    lib.mckg_detect_shared_host.argtypes = [ctypes.POINTER(Trace), vp, u64, ctypes.POINTER(u64),
                                            vp, ctypes.POINTER(u32)]
    lib.mckg_sort_triples.argtypes = [vp, u64, u32, vp, vp]
    lib.mckg_scan_stuck.argtypes = [vp, u32, u32, u32, vp, vp, vp, vp]
    lib.mckg_gen_c3.argtypes = [vp, vp, u32, u32, u64, vp]
    lib.mckg_gen_c5.argtypes = [vp, u32, u32, u32, u64, vp]
    lib.mckg_partition_global.argtypes = [vp, u64, u32, u64, vp, vp, vp]
    lib.mckg_detect_global.argtypes = [vp, u64, u64, vp, u64, vp, vp, vp, vp]
    lib.mckg_comm_init.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    lib.mckg_comm_destroy.argtypes = [vp]
    lib.mckg_comm_destroy.restype = None
    lib.mckg_detect_shared_mgpu.argtypes = [vp, ctypes.POINTER(Trace), ctypes.POINTER(RaceOut), vp]
    lib.mckg_detect_global_mgpu.argtypes = [vp, vp, u64, u64, vp, u64, vp, vp, vp, vp]
    _lib = lib
    return lib


def check(rc, what):
    if rc != MCKG_OK:
        msg = load().mckg_last_error().decode(errors="replace")
        raise MckgError(f"{what} failed with status {rc}: {msg}")
    return rc


def launch_stats():
    s = LaunchStats()
    load().mckg_get_launch_stats(ctypes.byref(s))
    return s
