"""The reference's own RunResult for every program of
tests/global_check_programs.py (the option-off baseline): run here, where
/root/reference exists:  python tests/make_global_check_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_bind as ob  # noqa: E402
from global_check_programs import PROGRAMS  # noqa: E402
from program_corpus import project  # noqa: E402


def main():
    gold = {name: project(ob.ref_run(src, filename="g.cu", capture=False)) for name, (src, _) in PROGRAMS.items()}
    with open(os.path.join(HERE, "golden", "global_check.json"), "w") as f:
        json.dump(gold, f, separators=(",", ":"), sort_keys=True)
    print(json.dumps({k: (v["exit"], v["diags"]) for k, v in gold.items()}))


if __name__ == "__main__":
    main()
