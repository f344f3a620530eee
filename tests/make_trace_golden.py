"""Golden --trace line streams (Machine::trace: stream dispatches, barrier
rules, grid completion) from the reference itself (oracle/_ref, this
container only), for the trace parity test (tests/test_gpu_trace.py).
Run: python tests/make_trace_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_bind as ob  # noqa: E402
from program_corpus import corpus  # noqa: E402

MAX_LINES = 4000


def pick(names):
    fixed = [n for n in names if n.startswith(("fig1", "scaled", "divbar"))]
    rest = [n for n in names if n.startswith(("conc", "rich", "rand", "num"))]
    return fixed + [n for i, n in enumerate(rest) if i % 7 == 0]


def main():
    progs = {n: (f, s) for n, f, s in corpus()}
    gold = json.load(open(os.path.join(HERE, "golden", "programs.json")))
    out = {}
    for n in pick(sorted(n for n in progs if n in gold)):
        f, s = progs[n]
        r = ob.ref_run(s, f, capture=False, trace=True)
        tr = r.get("trace", [])
        if 0 < len(tr) <= MAX_LINES:
            out[n] = tr
    path = os.path.join(HERE, "golden", "traces.json")
    json.dump(out, open(path, "w"), separators=(",", ":"))
    print(len(out), "programs,", sum(len(v) for v in out.values()), "lines ->", path)


if __name__ == "__main__":
    main()
