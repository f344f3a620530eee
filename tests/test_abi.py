"""The C-ABI library loads and exports every entry point include/mckg.h declares
(no compute calls: runs on CPU)."""
import ctypes
import os
import re

from paper_1211_6193_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mckg.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(mckg?_\w+)\(", src, re.M)))


def test_header_declares_the_exports():
    assert declared_symbols() == sorted(_abi.EXPORTS)


def test_library_exports_every_symbol():
    lib = _abi.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.mckg_abi_version() == 1


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_abi.Trace) == 48
    assert ctypes.sizeof(_abi.RaceOut) == 40
    assert ctypes.sizeof(_abi.LaunchStats) == 16


def test_errors_are_codes_not_exceptions():
    lib = _abi.load()
    assert lib.mckg_detect_shared(None, None, None) == _abi.MCKG_E_ARG
    assert b"null" in lib.mckg_last_error()
    assert lib.mckg_scan_stuck(None, 0, 0, 0, None, None, None, None) == _abi.MCKG_E_ARG
