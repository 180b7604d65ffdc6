"""Per-kernel share of device time from an ncu launch list
(ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...):
  python tools/launch_shares.py X.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", "")) * scale[r[iu]]
    except (ValueError, KeyError):
        continue
    name = r[ik].split("(")[0].replace("void ", "")
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{sum(cnt.values())} launches, {T * 1e3:.3f} ms total")
for k, v in tot.most_common():
    print(f"  {k:40s} {cnt[k]:5d} launches {v * 1e3:10.3f} ms {100 * v / T:6.2f} %")
