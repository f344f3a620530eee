"""Full-size BASELINE configs 2 and 4 through the whole checker on one B200
(host interpreter + K1 grid engine).  Prints one JSON line per run with the
outcome checks against the closed-form goldens."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1211_6193_b200 import checker  # noqa: E402
import gen_programs as gp  # noqa: E402


def c4_expected(nb, nt, seed):
    a = 2 * seed + 3
    dl = {}
    for b in range(nb):
        vals = []
        for t in range(nt):
            i = b * nt + t
            vals.append(2 * i if b % 3 == 0 else 2 * i + 1 if b % 3 == 1 else (i * a + b) % 7)
        odd = [t for t, v in enumerate(vals) if v % 2]
        if odd and len(odd) != nt:
            dl[b] = odd
    return dl


def run(name, src, **kw):
    t = time.time()
    r = checker.run_source(src, name + ".cu", step_limit=8_000_000_000, **kw)
    dt = time.time() - t
    return r, dt


which = sys.argv[1:] or ["c2", "c2racy", "c4"]
n = 1 << 24
for w in which:
    if w == "c2":
        r, dt = run("c2", gp.scaled(n, 256))
        ok = r["output"] == "OUTPUT: 830472184\n" and r["exit"] == 0
    elif w == "c2racy":
        r, dt = run("c2r", gp.scaled(n, 256, racy=True))
        ok = r["exit"] == 1 and [d["msg"] for d in r["diags"]] == ["Possible race on shared device memory detected at c2r.cu:17."]
    elif w.startswith("c4"):
        nb = int(os.environ.get("C4_BLOCKS", 1 << 16))
        r, dt = run("c4", gp.divergent_barrier_gen(nb, 1024, 0))
        exp = c4_expected(nb, 1024, 0)
        got = {s["bid"]: s["waiting"] for s in r["stuck_reports"] if s["kind"] == "barrier"}
        ok = r["exit"] == 3 and got == exp
    st = r.get("stats", {})
    print(json.dumps({"config": w, "ok": ok, "wall_s": dt, "exit": r.get("exit"), "engine_error": r.get("engine_error"),
                      "steps": r.get("steps"), "stats": st, "n_reported": len(r.get("reported", [])),
                      "diags": [d["msg"] for d in r.get("diags", [])][:4],
                      "device_steps_per_s": st.get("device_steps", 0) / max(1e-9, st.get("grid_ms", 0) / 1e3)}),
          flush=True)
