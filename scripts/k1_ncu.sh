cat > /tmp/k1prof.py <<'PY'
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_1211_6193_b200 import checker
import gen_programs as gp
r = checker.run_source(gp.scaled(1 << 18, 256), "c2s.cu", step_limit=8_000_000_000)
print(r["exit"], r["stats"]["grid_ms"])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -c 1 -o gpurun_out/prof_k1b python /tmp/k1prof.py > gpurun_out/ncu_k1b.log 2>&1; echo "ncu rc=$?"
