"""Per-iteration cost of the distributed protocol on the north-star fixed-work
workload (f2 d=8 rtol 1e-6, 64-subdomain init, fixed iterations), on one GPU:

  * P = 1: run_distributed(backend="nccl") on a 1-rank NCCL group vs the
    native integrate() loop (same region sets; the difference is the protocol:
    record all-gather, status reads, Python planning);
  * P = 2, 4, 8: run_distributed(backend="concurrent") - one thread per rank,
    every rank's store on this GPU, device-tensor transfers - vs integrate()
    on the same GPU: the GPU work is the same (the rank stores partition the
    same region set) and serialises on one device, so the excess over
    integrate() is the P-rank protocol (barriers, record exchange, planning,
    K4/K5 transfers), an upper bound on what P GPUs would pay per iteration.

Per-iteration cost = slope of the excess between two run lengths (so the
per-run setup - communicator, first allocations, settle - is not spread over
the iterations).  Prints one JSON line per P (medians of 3) and the projected
P-GPU speed-up T1 / (T1 / P + its * excess_P).
  python tools/probe_protocol.py [iterations] [short iterations]"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2511_01573_b200 as hb

its = int(sys.argv[1]) if len(sys.argv) > 1 else 22
its0 = int(sys.argv[2]) if len(sys.argv) > 2 else 12
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
f = hb.make_integrand("f2", 8)
dom = hb.HyperRect.unit_cube(8)
cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


# warm-up (allocator, library, kernels)
hb.integrate(f, dom, cfg, initial_regions=64)
rows = []
for P in (1, 2, 4, 8):
    rc = hb.RedistributionConfig(initial_subdomains_per_rank=64 // P)
    backend = "nccl" if P == 1 else "concurrent"
    res = {}
    for n_it in (its0, its):
        c = hb.DriverConfig(1e-6, max_iterations=n_it, max_regions=1 << 40)
        t_nat, t_dist = [], []
        for rep in range(4):
            a, r = timed(lambda: hb.integrate(f, dom, c, initial_regions=64))
            b, dr = timed(lambda: hb.run_distributed(f, dom, c, rc, workers=P, backend=backend))
            if rep:
                t_nat.append(a)
                t_dist.append(b)
        assert dr.result.total_f_evals == r.total_f_evals and dr.result.iterations == r.iterations
        res[n_it] = (statistics.median(t_nat), statistics.median(t_dist), r, dr)
    tn, td, r, dr = res[its]
    excess = ((td - tn) - (res[its0][1] - res[its0][0])) / (its - its0)
    rows.append(dict(P=P, backend=backend, iterations=its, evals=r.total_f_evals, integrate_s=tn, distributed_s=td,
                     per_run_excess_s=(td - tn) - its * excess,
                     protocol_us_per_iteration=excess * 1e6,
                     same_integral=dr.result.integral == r.integral,
                     projected_speedup=tn / (tn / P + its * max(excess, 0.0)),
                     messages=dr.messages_total, regions_transferred=dr.regions_transferred_total))
    print(json.dumps(rows[-1]), flush=True)
dist.destroy_process_group()
