"""Summarise an ncu --set full capture of k1_gm_eval into JSON (profiles/).
usage: python tools/ncu_summary.py <report.ncu-rep> <regions_in_launch> <evals_per_region> <out.json>"""
import collections
import csv
import io
import json
import subprocess
import sys

rep, regions, K, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = lambda k: float(vals[hdr.index(k)].replace(",", ""))  # noqa: E731
unit = lambda k: units[hdr.index(k)]  # noqa: E731
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}
t = get("gpu__time_duration.sum") * scale[unit("gpu__time_duration.sum")]
rd = get("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
wr = get("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
sh = srows[1]
iE, iS = sh.index("Instructions Executed"), sh.index("Source")
ops = collections.Counter()
for r in srows[2:]:
    try:
        n = int(r[iE])
    except (ValueError, IndexError):
        continue
    op = r[iS].strip().split()
    if op:
        ops[(op[1] if op[0].startswith("@") else op[0]).split(".")[0]] += n
warps = regions / 32.0
dp = sum(ops[k] for k in ("DFMA", "DADD", "DMUL"))
doc = {
    "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "k1_gm_eval",
    "regions_in_launch": regions, "evals_per_region": K,
    "duration_s": t, "evals_per_s": regions * K / t,
    "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
    "dram_bytes_per_region": (rd + wr) / regions,
    "algorithmic_bytes_per_region": None,
    "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": get("launch__registers_per_thread"),
    "sm_clock_hz": get("sm__cycles_elapsed.avg.per_second") * 1e9,
    "warp_instructions_per_region": sum(ops.values()) / warps,
    "fp64_instructions_per_region": dp / warps, "fp64_instructions_per_eval": dp / warps / K,
    "sass_mix_per_region": {k: round(v / warps, 1) for k, v in ops.most_common(16)},
}
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc, indent=1))
