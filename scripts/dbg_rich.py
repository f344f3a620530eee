import os, sys; os.environ["MCK_DIAG_SWEEP"]="1"; sys.path.insert(0,"."); sys.path.insert(0,"tests")
import gen_programs as gp
from paper_1211_6193_b200 import checker
for s in [46, 22]:
    r = checker.run_source(gp.random_kernel2(s), f"rich{s}.cu")
    print(s, [(d["line"], d["sweep"], d["msg"][:40]) for d in r["diags"]], r["steps"])
