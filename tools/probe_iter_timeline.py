"""Per-iteration wall-time timeline of run_distributed (1 NCCL rank, one-sync
protocol) vs the native integrate loop on the north-star workload: where
(which iteration sizes) the distributed loop's excess appears.
  python tools/probe_iter_timeline.py [iterations]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200.worker import DeviceWorker

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29549")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 22
f = hb.make_integrand("f2", 8)
dom = hb.HyperRect.unit_cube(8)
cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)
rc = hb.RedistributionConfig(initial_subdomains_per_rank=64)
stamps = []
orig = DeviceWorker.evaluate_begin


def eb(self):
    stamps.append(time.perf_counter())
    return orig(self)


for rep in range(3):
    hb.integrate(f, dom, cfg, initial_regions=64)
    hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
DeviceWorker.evaluate_begin = eb
torch.cuda.synchronize()
t0 = time.perf_counter()
dr = hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
t1 = time.perf_counter()
DeviceWorker.evaluate_begin = orig
nat = []
st = {}
t2 = time.perf_counter()
r = hb.integrate(f, dom, cfg, initial_regions=64, trace=lambda tr: nat.append((time.perf_counter(), tr.active_regions)),
                 stats=st)
t3 = time.perf_counter()
d_dist = [b - a for a, b in zip(stamps, stamps[1:] + [t1])]
d_nat = [b[0] - a[0] for a, b in zip([(t2, 0)] + nat[:-1], nat)]
print(json.dumps({"dist_total_ms": 1e3 * (t1 - t0), "native_total_ms": 1e3 * (t3 - t2),
                  "native_device_ms": st, "dist_device_ms": dr.device_stats,
                  "per_iteration": [{"it": i + 1, "regions": n, "dist_us": round(1e6 * a), "native_us": round(1e6 * b)}
                                    for i, (a, b, (_, n)) in enumerate(zip(d_dist, d_nat, nat))]}, indent=0))
dist.destroy_process_group()
