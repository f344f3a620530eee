"""K1 experiment: C2 (scaled Fig. 1, 256-thread blocks) grid time per
multiplexing factor K (run once per MCKG_K1_K value: it is read at load)."""
import json, os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_1211_6193_b200 import checker
import gen_programs as gp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
src = gp.scaled(n, 256)
k = os.environ.get("MCKG_K1_K", "auto")
if True:
    for rep in range(2):
        r = checker.run_source(src, "c2.cu", step_limit=8_000_000_000)
        st = r["stats"]
        print(json.dumps({"K": k, "n": n, "out": r["output"].strip(), "grid_ms": st["grid_ms"],
                          "steps_per_s": st["device_steps"] / st["grid_ms"] * 1e3,
                          "launches": st["kernel_launches"], "err": r.get("engine_error")}), flush=True)
