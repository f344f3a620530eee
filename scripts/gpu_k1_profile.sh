#!/bin/bash
# Full-size C2 racy + C4 through the checker, and one ncu capture of K1.
mkdir -p gpurun_out
python scripts/gpu_fullsize.py c2racy c4 > gpurun_out/full2.log 2>&1; echo "full rc=$?"
cat gpurun_out/full2.log
cat > /tmp/k1prof.py <<'PY'
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_1211_6193_b200 import checker
import gen_programs as gp
r = checker.run_source(gp.scaled(1 << 20, 256), "c2s.cu", step_limit=8_000_000_000)
print(r["exit"], r["output"], r["stats"])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -c 1 \
  -o gpurun_out/prof_k1 python /tmp/k1prof.py > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_k1.log
