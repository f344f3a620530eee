#!/bin/bash
# ncu --set full of K1 on C2 scaled to 2^18 ints (1024 blocks x 256 threads):
# grid_kernel<1> and tail_kernel; summaries into gpurun_out/
mkdir -p gpurun_out
cat > /tmp/k1prof.py <<'PY'
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_1211_6193_b200 import checker
import gen_programs as gp
r = checker.run_source(gp.scaled(1 << 18, 256), "c2s.cu", step_limit=8_000_000_000)
print(r["exit"], r["stats"]["grid_ms"])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_kernel|tail_kernel" -c 2 -o gpurun_out/prof_k1 python /tmp/k1prof.py > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_k1.ncu-rep 25 > gpurun_out/k1_ncu_summary.txt 2>&1
