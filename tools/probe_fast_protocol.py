"""Host-side cost of one iteration of run_distributed's one-sync protocol
(1 NCCL rank, f2 d=8 init 64): every libhcub call is timed (ctypes wall,
includes the GPU work it waits for), the rest is Python.  Compared with the
native integrate loop on the same workload.
  python tools/probe_fast_protocol.py [iterations]"""
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200 import _lib

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29547")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 16
f = hb.make_integrand("f2", 8)
dom = hb.HyperRect.unit_cube(8)
cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)
rc = hb.RedistributionConfig(initial_subdomains_per_rank=64)
L = _lib.lib()
T, N = collections.Counter(), collections.Counter()
for name in _lib.SIGNATURES:
    fn = getattr(L, name)

    def w(*a, _f=fn, _n=name):
        t0 = time.perf_counter()
        try:
            return _f(*a)
        finally:
            T[_n] += time.perf_counter() - t0
            N[_n] += 1
    setattr(L, name, w)
for rep in range(3):
    hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
    hb.integrate(f, dom, cfg, initial_regions=64)
T.clear(); N.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
dr = hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
t1 = time.perf_counter()
lib_s = sum(T.values())
calls = {k: [N[k], round(1e6 * v / N[k], 1)] for k, v in sorted(T.items(), key=lambda kv: -kv[1])}
T.clear(); N.clear()
torch.cuda.synchronize()
t2 = time.perf_counter()
r = hb.integrate(f, dom, cfg, initial_regions=64)
t3 = time.perf_counter()
st = dr.device_stats
dev_us = 1e3 * (st["k1_ms"] + st["k2_ms"] + st["k3_ms"]) / its
print(json.dumps({"iterations": its, "distributed_us_per_it": 1e6 * (t1 - t0) / its,
                  "integrate_us_per_it": 1e6 * (t3 - t2) / its,
                  "excess_us_per_it": 1e6 * ((t1 - t0) - (t3 - t2)) / its,
                  "device_k1_k2_k3_us_per_it": dev_us,
                  "python_us_per_it": 1e6 * ((t1 - t0) - lib_s) / its,
                  "lib_calls_us": calls, "same_integral": r.integral == dr.result.integral}, indent=1))
dist.destroy_process_group()
if len(sys.argv) > 2:  # python-side profile of the loop (cProfile, by own time)
    import cProfile
    import io
    import pstats
    dist.init_process_group("nccl", rank=0, world_size=1)
    hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(45)
    print(s.getvalue())
    dist.destroy_process_group()
