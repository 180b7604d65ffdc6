"""Summarise an ncu --set full capture of k1_gm_eval into JSON (profiles/).
usage: python tools/ncu_summary.py <report.ncu-rep> <regions_in_launch> <evals_per_region> <out.json> [note]

algorithmic bytes per region of the fused-split K1 at dimension d (unique
bytes that must cross HBM): parent box 2*d*8 B shared by its two children,
child box written 2*d*8 B, survivor index 8 B and parent axis 1 B per parent
pair, outputs integral/error/volume/split-extent 4*8 B + axis 1 B."""
import collections
import csv
import io
import json
import subprocess
import sys

rep, regions, K, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
note = sys.argv[5] if len(sys.argv) > 5 else ""
D = {33: 3, 93: 5, 149: 6, 401: 8, 1245: 10}.get(K)
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
    "algorithmic_bytes_per_region": (2 * D * 8 / 2 + 2 * D * 8 + 9 / 2 + 4 * 8 + 1) if D else None,
    "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": get("launch__registers_per_thread"),
    "sm_clock_hz": get("sm__cycles_elapsed.avg.per_second") * 1e9,
    "warp_instructions_per_region": sum(ops.values()) / warps,
    "fp64_instructions_per_region": dp / warps, "fp64_instructions_per_eval": dp / warps / K,
    "sass_mix_per_region": {k: round(v / warps, 1) for k, v in ops.most_common(16)},
}
stalls = {x[len("smsp__pcsamp_warps_issue_stalled_"):]: get(x) for x in hdr
          if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("_not_issued")}
tot = sum(stalls.values()) or 1
doc["stall_samples_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda t: -t[1])
                            if v / tot > 0.005}
if note:
    doc["note"] = note
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc, indent=1))
