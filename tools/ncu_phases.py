"""Per-loop breakdown of an ncu source page (SASS): warp instructions
executed, FP64 share and stall samples for every backward-branch loop.
  python tools/ncu_phases.py gpurun_out/<name>.ncu-rep [min_share]"""
import csv
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, isamp, iexe = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                 "Instructions Executed"))
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
ir = [hdr.index(k) for k in reasons]
ins = []
stalls = []
for r in rows[2:]:
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), float(r[isamp] or 0), float(r[iexe] or 0)))
        stalls.append([float(r[i] or 0) for i in ir])
    except (ValueError, IndexError):
        pass
base = ins[0][0]
tot_s = sum(x[2] for x in ins)
tot_e = sum(x[3] for x in ins)
print(f"total warp instructions {tot_e:.4g}, samples {tot_s:.0f}")
idx = {a: i for i, (a, *_ ) in enumerate(ins)}
loops = []
for i, (a, src, s, e) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", src)
    if m and m.group(1):
        t = int(m.group(1), 16) + base if int(m.group(1), 16) < base else int(m.group(1), 16)
        if t < a and t in idx:
            loops.append((idx[t], i))
minshare = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for lo, hi in loops:
    body = ins[lo:hi + 1]
    s = sum(x[2] for x in body)
    e = sum(x[3] for x in body)
    dp = sum(x[3] for x in body if re.match(r"(@!?U?P\d+\s+)?D(FMA|ADD|MUL)\b", x[1]))
    if s / tot_s >= minshare:
        print(f"loop {body[0][0]-base:#x}-{body[-1][0]-base:#x} ({len(body)} instrs): samples {100*s/tot_s:5.1f} %, "
              f"warp insts {100*e/tot_e:5.1f} %, DP/inst {dp/max(e,1):.2f}")
        agg = [sum(st[k] for st in stalls[lo:hi + 1]) for k in range(len(reasons))]
        tot = sum(agg) or 1
        print("    " + ", ".join(f"{reasons[k][6:]} {100*agg[k]/tot:.0f}%" for k in sorted(range(len(reasons)), key=lambda k: -agg[k])
                                  if agg[k] / tot > 0.02))
