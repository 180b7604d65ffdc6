"""Per-instruction stall attribution from an ncu --set full report (SASS
source page): total samples, the instructions with the most long-scoreboard
and barrier stalls, and samples / executions per opcode.
  python tools/ncu_sass_stalls.py <report.ncu-rep>"""
import collections
import csv
import io
import subprocess
import sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


S = "Warp Stall Sampling (All Samples)"
tot = sum(f(r[ix[S]]) for r in data)
cols = [k for k in h if k.startswith("stall_")]
print(f"total samples {tot:.0f}")
for k in sorted(cols, key=lambda k: -sum(f(r[ix[k]]) for r in data))[:10]:
    print(f"  {k:24s} {100 * sum(f(r[ix[k]]) for r in data) / tot:5.1f} %")
for col in ("stall_long_sb", "stall_barrier", "stall_wait"):
    print(f"-- top {col}")
    for r in sorted(data, key=lambda r: -f(r[ix[col]]))[:8]:
        print(f"   {r[0]} {r[1][:70]:70s} {f(r[ix[col]]):8.0f}")
c, n = collections.Counter(), collections.Counter()
for r in data:
    toks = r[1].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    c[op] += f(r[ix[S]])
    n[op] += f(r[ix["Instructions Executed"]])
print("-- opcode: samples share, warp instructions executed")
for k, v in c.most_common(18):
    print(f"   {k:10s} {100 * v / tot:5.1f} %  {n[k]:.3e}")
