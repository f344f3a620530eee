"""Generates tests/golden/edge_programs.json: the reference itself
(oracle/_ref/libmckref.so, Machine::run, round robin) on every program of
tests/edge_programs.py.  Run here, where /root/reference exists:
    python tests/make_edge_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_bind as ob  # noqa: E402
from edge_programs import edge_cases  # noqa: E402
from program_corpus import project  # noqa: E402


def main():
    assert ob.ref() is not None, "oracle/_ref/libmckref.so missing: build the oracle first"
    gold = {}
    for name, (fname, limit, src) in sorted(edge_cases().items()):
        if isinstance(limit, tuple):  # ("T", d): the unlimited total + d
            total = ob.ref_run(src, filename=fname, step_limit=10**12, capture=False)["steps"]
            limit = total + limit[1]
        r = ob.ref_run(src, filename=fname, policy="rr", step_limit=limit, capture=False)
        gold[name] = {"fname": fname, "step_limit": limit, "src": src, "gold": project(r)}
    path = os.path.join(HERE, "golden", "edge_programs.json")
    with open(path, "w") as f:
        json.dump(gold, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {len(gold)} edge golden runs to {path}")


if __name__ == "__main__":
    main()
