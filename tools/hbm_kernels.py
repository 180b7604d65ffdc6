"""Largest launch per kernel from an ncu metrics CSV
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv):
DRAM bytes / duration vs MEASURED_PEAKS.json hbm_gbs.
  python tools/hbm_kernels.py launches.csv out.json"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iid, ik, im, iu, iv = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "second": 1.0}
launch = collections.defaultdict(dict)
for r in rows[1:]:
    launch[r[iid]]["name"] = r[ik].split("(")[0].replace("void ", "").split("<")[0]
    launch[r[iid]][r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
best = {}
for L in launch.values():
    b = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
    t = L.get("gpu__time_duration.sum", 0)
    n = L["name"]
    if t and (n not in best or b > best[n]["bytes"]):
        best[n] = {"bytes": b, "seconds": t, "GBps": b / t / 1e9, "frac_of_measured_hbm": b / t / 1e9 / peak}
doc = {"note": f"largest launch per kernel (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
               f"dram__bytes_write.sum --clock-control none: serialised, cold cache) of tools/profile_store.py; "
               f"frac vs MEASURED_PEAKS.json hbm_gbs={peak}", "kernels": best}
json.dump(doc, open(sys.argv[2], "w"), indent=1)
for n, v in sorted(best.items(), key=lambda kv: -kv[1]["bytes"]):
    print(f"{n:20s} {v['bytes'] / 1e6:10.1f} MB {v['seconds'] * 1e3:8.3f} ms {v['GBps']:8.1f} GB/s {v['frac_of_measured_hbm']:.2f}")
