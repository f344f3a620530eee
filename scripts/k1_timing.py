"""K1 timing probe: scaled Fig. 1 at 2^20 (4096 blocks) and C4 at 1024 blocks."""
import json, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_1211_6193_b200 import checker
import gen_programs as gp
for name, src in [("c2_4096", gp.scaled(1 << 20, 256)), ("c4_1024", gp.divergent_barrier_gen(1024, 1024, 0))]:
    t = time.time()
    r = checker.run_source(src, name + ".cu", step_limit=8_000_000_000)
    st = r["stats"]
    print(json.dumps({"name": name, "exit": r["exit"], "wall": time.time() - t, "grid_ms": st["grid_ms"],
                      "steps_per_s": st["device_steps"] / st["grid_ms"] * 1e3,
                      "block_sweeps": st["block_sweeps"], "solo_sweeps": st["solo_sweeps"],
                      "block_cycles": st["block_cycles"], "solo_cycles": st["solo_cycles"],
                      "err": r.get("engine_error")}), flush=True)
