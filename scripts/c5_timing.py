"""K6 timing probe: mckg_detect_global on C5 (2^29 records = one GPU's share of configs[4]) per route."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1211_6193_b200 import _abi, global_race as gr
blocks = int(__import__("os").environ.get("C5_BLOCKS", 1 << 17))
ev = gr.gen_c5(0, blocks, blocks, device="cuda")
lib = _abi.load()
s = torch.cuda.current_stream()
for name, dbg in [(r, {"tile": 0, "buckets": 256}[r]) for r in (sys.argv[1:] or ["tile", "buckets", "tile"])]:
    lib.mckg_set_debug(dbg)
    out = gr.GlobalOut(ev.shape[0] // 8)
    for i in range(int(__import__("os").environ.get("C5_REPS", "6"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        e0.record(s)
        gr.detect(ev, 0, out.reset(), s)
        e1.record(s)
        torch.cuda.synchronize()
        print(name, i, f"event {e0.elapsed_time(e1):.3f} ms wall {1e3 * (time.perf_counter() - t):.3f} ms",
              int(out.n.item()), int(out.status.item()), flush=True)
lib.mckg_set_debug(0)
