cat > /tmp/m.py <<'PY'
import sys, torch; sys.path.insert(0,'.')
from paper_1211_6193_b200 import race, _abi
ev, bs = race.gen_c3(0, 1<<20)
tr = race.make_trace(ev, bs, 4096, max_block_events=1024)
out = race.RaceOut(1<<27)
st = torch.zeros(4, dtype=torch.int32, device='cuda')
out._c.status = st.data_ptr()
out.reset(); race.detect_shared_async(tr, out, reset=False); torch.cuda.synchronize()
print("racing X", st[1].item(), "candidates", st[2].item(), "triples", out.n_triples.item())
PY
MCKG_DEBUG=12 python /tmp/m.py
for d in 0 4; do echo "debug=$d"; MCKG_DEBUG=$d python bench.py --steps 30 --warmup 3 --no-cpu --e2e-blocks 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'])"; done
