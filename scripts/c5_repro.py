import sys
sys.path.insert(0, ".")
import torch
from paper_1211_6193_b200 import _abi, global_race as gr
blocks = int(sys.argv[1])
dbg = int(sys.argv[2])
ev = gr.gen_c5(0, blocks, blocks, device="cuda")
lib = _abi.load(); lib.mckg_set_debug(dbg)
out = gr.GlobalOut(ev.shape[0] // 8)
gr.detect(ev, 0, out.reset(), torch.cuda.current_stream())
torch.cuda.synchronize()
print(blocks, dbg, int(out.n.item()), int(out.status.item()), flush=True)
