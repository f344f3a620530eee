"""Summarise an ncu report: key raw metrics + top source lines by stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
flt = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []  # one kernel of a multi-kernel report
raw = subprocess.run(["ncu", "-i", rep, *flt, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2] if len(r) > 2 else r[1]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]
for k, x in zip(h, v):
    if k in want or (k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
                     and float(x or 0) > 0.2):
        print(f"{k:80s} {x}")
src = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, out = None, []
for row in csv.reader(src.splitlines()):
    if len(row) == 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if len(row) < 8 or row[0] in ("Line No", ""):
        continue
    try:
        out.append((int(row[7]), int(row[4]), fname, row[0], row[1][:80]))
    except ValueError:
        pass
tot, stt = sum(o[0] for o in out), sum(o[1] for o in out)
print(f"warp instructions {tot}  stall samples {stt}")
for o in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{o[0]:>11} {o[1]:>7} {o[2]}:{o[3]} {o[4]}")
