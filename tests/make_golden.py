"""Generates tests/golden/programs.json by running every corpus program through
the reference checker itself (oracle/_ref/libmckref.so: /root/reference/proj
built by oracle/Makefile) under the round-robin schedule.  Run here, where
/root/reference exists:  python tests/make_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_bind as ob  # noqa: E402
from program_corpus import corpus, host_corpus, project, HOST_STEP_LIMIT, FRONTEND_CASES  # noqa: E402


def main():
    assert ob.ref() is not None, "oracle/_ref/libmckref.so missing: build the oracle first"
    gold = {}
    for name, fname, src in corpus():
        r = ob.ref_run(src, filename=fname, policy="rr", capture=False)
        gold[name] = project(r)
    path = os.path.join(HERE, "golden", "programs.json")
    with open(path, "w") as f:
        json.dump(gold, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {len(gold)} golden runs to {path}")
    # the reference's DEFAULT schedule (seeded random, seed 0) on the BASELINE
    # program families: SURVEY F4 says it agrees with round-robin there
    seed0 = {}
    for name, fname, src in corpus():
        if name.startswith(("fig1", "scaled", "divbar")):
            seed0[name] = project(ob.ref_run(src, filename=fname, policy="random", seed=0, capture=False))
    with open(os.path.join(HERE, "golden", "programs_seed0.json"), "w") as f:
        json.dump(seed0, f, separators=(",", ":"), sort_keys=True)
    host = {}
    for name, fname, src in host_corpus():
        r = ob.ref_run(src, filename=fname, policy="rr", capture=False, step_limit=HOST_STEP_LIMIT)
        host[name] = project(r)
    for name, src in FRONTEND_CASES.items():
        r = ob.ref_run(src, filename=name + ".cu", policy="rr", capture=False)
        host["fe_" + name] = {"frontend_error": r.get("frontend_error"), "line": r.get("line"),
                              "exit": r.get("exit")}
    path = os.path.join(HERE, "golden", "host_programs.json")
    with open(path, "w") as f:
        json.dump(host, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {len(host)} golden host runs to {path}")


if __name__ == "__main__":
    main()
