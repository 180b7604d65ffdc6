"""Key K1 counters + stall breakdown from an ncu --set full report:
  python tools/ncu_stalls.py gpurun_out/<name>.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
get = {x: (v[i], u[i]) for i, x in enumerate(h)}
for k in ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed.sum", "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
          "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]:
    if k in get:
        print(f"{k:70s} {get[k][0]} {get[k][1]}")
tot = 0
st = {}
for x in h:
    if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("_not_issued"):
        st[x[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(get[x][0].replace(",", ""))
tot = sum(st.values())
for k, c in sorted(st.items(), key=lambda t: -t[1]):
    if c / tot > 0.005:
        print(f"  stall {k:28s} {100 * c / tot:5.1f} %")
