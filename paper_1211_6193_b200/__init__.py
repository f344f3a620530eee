"""paper_1211_6193_b200 -- B200-native data-parallel core of the arXiv 1211.6193
CUDA-C checker (reference: minicudak, /root/reference/proj).

Hot path, hand-written sm_100a kernels in ``csrc/`` behind the
C ABI ``include/mckg.h`` (``libmckg.so``): the grid interpreter with its fused
race shadow and deadlock scan (K1, ``interp.cu``, incl. the serial-tail kernel
and the GPU exhaustive-interleaving oracle K7), shared-memory race detection
over access traces (K2, ``detect.cu``), the barrier-deadlock scan (K4,
``stuck.cu``), cross-block global races (K3/K6, ``global_race.cu``), report
compaction and the radix sort (``sort.cu``), the NCCL exchange steps
(``mgpu.cu``).  The C++ host checker (``host/``) mirrors the reference's
``mck::`` API.  torch is used for device memory and streams only; there is no
CPU fallback.
"""
import importlib

from . import _abi  # noqa: F401

__all__ = ["_abi", "race"]


def __getattr__(name):
    if name == "race":
        return importlib.import_module(".race", __name__)
    raise AttributeError(name)
