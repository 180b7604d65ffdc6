"""Where the distributed loop's per-iteration host time goes (1 rank, NCCL):
wraps the worker / transport calls of run_distributed with wall-clock timers."""
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200 import distributed as D
from paper_2511_01573_b200.worker import DeviceWorker

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29535")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
T = collections.Counter()
N = collections.Counter()


def wrap(cls, name):
    fn = getattr(cls, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            T[name] += time.perf_counter() - t0
            N[name] += 1
    setattr(cls, name, w)


for n in ("evaluate_begin", "evaluate_end", "classify", "append", "take_top_device"):
    wrap(DeviceWorker, n)
for n in ("allgather_rows", "allgather_ints", "exchange", "complete"):
    wrap(D._TorchTransport, n)
from paper_2511_01573_b200 import _lib
L = _lib.lib()
for cname in ("hcub_worker_classify", "hcub_worker_evaluate_end", "hcub_worker_size"):
    cfn = getattr(L, cname)

    def cw(*a, _f=cfn, _n=cname):
        t0 = time.perf_counter()
        try:
            return _f(*a)
        finally:
            T[_n] += time.perf_counter() - t0
            N[_n] += 1
    setattr(L, cname, cw)
f = hb.make_integrand("f2", 8)
dom = hb.HyperRect.unit_cube(8)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 18
cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)
rc = hb.RedistributionConfig(initial_subdomains_per_rank=64)
hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
T.clear(); N.clear()
t0 = time.perf_counter()
dr = hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
tot = time.perf_counter() - t0
st = dr.device_stats
print(json.dumps({"iterations": its, "total_ms": 1e3 * tot, "device_k1_k2_k3_ms": [st["k1_ms"], st["k2_ms"], st["k3_ms"]],
                  "calls_ms": {k: round(1e3 * v, 3) for k, v in T.items()}, "counts": dict(N)}, indent=1))
import cProfile
import io
import pstats
pr = cProfile.Profile()
pr.enable()
hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue())
dist.destroy_process_group()
