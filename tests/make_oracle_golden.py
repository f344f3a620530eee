"""Generates tests/golden/oracle.json: the reference's oracleRace
(oracle/_ref/libmckref.so) on every program of tests/oracle_programs.py.
Run here, where /root/reference exists:  python tests/make_oracle_golden.py"""
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_bind as ob  # noqa: E402
from oracle_programs import PROGRAMS  # noqa: E402


def ref_oracle(src, o):
    lib = ob.ref()
    lib.mckref_oracle.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_void_p)]
    out = ctypes.c_void_p()
    lib.mckref_oracle(src.encode(), b"o.cu", o["max_interleavings"], o["max_threads"], o["max_accesses"],
                      ctypes.byref(out))
    s = ctypes.string_at(out.value).decode()
    lib.mckref_free(out)
    return json.loads(s)


def main():
    gold = {name: ref_oracle(src, o) for name, (src, o) in PROGRAMS.items()}
    with open(os.path.join(HERE, "golden", "oracle.json"), "w") as f:
        json.dump(gold, f, indent=0, sort_keys=True)
    for k, v in gold.items():
        print(k, v)


if __name__ == "__main__":
    main()
