"""paper_1211_6193_b200 -- B200-native data-parallel core of the arXiv 1211.6193
CUDA-C checker (reference: minicudak, /root/reference/proj).

Hot path: shared-memory race detection (K2), barrier-deadlock
classification (K4) and report ordering (K5) as hand-written sm_100a kernels in
``csrc/``, behind the C ABI ``include/mckg.h`` (``libmckg.so``).  torch is used
for device memory and streams only.  There is no CPU fallback.
"""
import importlib

from . import _abi  # noqa: F401

__all__ = ["_abi", "race"]


def __getattr__(name):
    if name == "race":
        return importlib.import_module(".race", __name__)
    raise AttributeError(name)
