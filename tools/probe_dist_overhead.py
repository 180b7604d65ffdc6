"""Per-iteration host overhead of run_distributed (NCCL transport, 1 rank)
vs the fully native integrate loop, on the bench workload."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2511_01573_b200 as hb

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
f = hb.make_integrand("f2", 8)
dom = hb.HyperRect.unit_cube(8)
for its in (12, 20, 26):
    cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = hb.integrate(f, dom, cfg, initial_regions=64)
        t1 = time.perf_counter()
        dr = hb.run_distributed(f, dom, cfg, hb.RedistributionConfig(initial_subdomains_per_rank=64), workers=1,
                                backend="nccl")
        torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps(dict(iterations=its, integrate_s=t1 - t0, distributed_s=t2 - t1,
                          overhead_per_iter_ms=1e3 * ((t2 - t1) - (t1 - t0)) / its, same=r.integral == dr.result.integral,
                          stats=dr.device_stats)), flush=True)
dist.destroy_process_group()
