"""Host-side profile (cProfile) of run_distributed's per-iteration protocol
on one rank (NCCL process group of size 1), f2 d=8 init 64, 20 iterations."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2511_01573_b200 as hb

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29534")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
f = hb.make_integrand("f2", 8)
dom = hb.HyperRect.unit_cube(8)
its = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)
rc = hb.RedistributionConfig(initial_subdomains_per_rank=64)
hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
pr = cProfile.Profile()
pr.enable()
hb.run_distributed(f, dom, cfg, rc, workers=1, backend="nccl")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
dist.destroy_process_group()
