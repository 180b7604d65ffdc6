"""Multi-GPU leg of bench.py (torchrun, one rank per GPU).

Strong scaling on the fixed-work workload: the 64 initial subdomains are
dealt round-robin over the ranks (initial_subdomains_per_rank = 64 / N, ref
distributed.py:371-378), so the global region set - and the total number of
integrand evaluations - is the same for every N; ranks rebalance with the
round-robin protocol over NCCL.  Time = max over ranks of the CUDA-event
time of one run_distributed call, each bracketed by a barrier and a device
synchronisation.
"""

from __future__ import annotations

import os
import time


def run_multi_gpu(args, rank, world, D, FN, TAU, INIT, F_FLOPS, peak, clock_sampler, traffic=None):
    import torch
    import torch.distributed as dist

    import paper_2511_01573_b200 as hb

    local = int(os.environ.get("LOCAL_RANK", rank))
    ngpu = torch.cuda.device_count()
    dev = local % max(ngpu, 1)
    torch.cuda.set_device(dev)
    hb.set_device(dev)
    # NCCL needs one GPU per rank; a 1-GPU box can still smoke-test the path
    backend = "nccl" if ngpu >= world else "gloo"
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        if INIT % world:
            raise ValueError(f"{INIT} initial subdomains do not split over {world} ranks")
        f = hb.make_integrand(FN, D)
        dom = hb.HyperRect.unit_cube(D)
        cfg = hb.DriverConfig(TAU, max_iterations=args.iterations, max_regions=1 << 40)
        rcfg = hb.RedistributionConfig(initial_subdomains_per_rank=INIT // world)

        def step():
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            dr = hb.run_distributed(f, dom, cfg, rcfg, workers=world, backend="nccl")
            e1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            dist.barrier()
            return dr, e0.elapsed_time(e1) * 1e-3, wall

        for _ in range(args.warmup):
            step()
        res = []
        with clock_sampler(dev) as clk:
            for _ in range(args.steps):
                res.append(step())
        dev_s = torch.tensor([sum(r[1] for r in res), sum(r[2] for r in res)], dtype=torch.float64,
                             device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(dev_s, op=dist.ReduceOp.MAX)
        t_dev, t_wall = dev_s.tolist()

        # time-to-tolerance of BASELINE configs[1] (f2 d=5 rtol 1e-6) through the
        # distributed engine with the reference's default 8 subdomains per rank
        f5 = hb.make_integrand("f2", 5)
        cfg5 = hb.DriverConfig(1e-6, max_regions=1 << 40)
        ttt = []
        for rep in range(4):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dr5 = hb.run_distributed(f5, hb.HyperRect.unit_cube(5), cfg5, hb.RedistributionConfig(), workers=world,
                                     backend="nccl")
            torch.cuda.synchronize()
            tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                              device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            if rep:
                ttt.append(tt.item())
        ttt.sort()

        # the rebalancing stress shapes of BASELINE configs[3] (f3 d=10, 80
        # initial subdomains) and configs[4] (f6 d=6, 48): round-robin
        # transfers are active, capped iterations keep each run short
        rebal = []
        for idx, fid, d, tau, init, its in ((3, "f3", 10, 1e-5, 80, 16), (4, "f6", 6, 1e-4, 48, 18)):
            per = init // world if init % world == 0 else 8
            rc = hb.RedistributionConfig(initial_subdomains_per_rank=per)
            cf = hb.DriverConfig(tau, max_iterations=its, max_regions=1 << 40)
            fx = hb.make_integrand(fid, d)
            times = []
            for rep in range(3):
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                drx = hb.run_distributed(fx, hb.HyperRect.unit_cube(d), cf, rc, workers=world, backend="nccl")
                torch.cuda.synchronize()
                tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                                  device="cuda" if backend == "nccl" else "cpu")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                if rep:
                    times.append(tt.item())
            t = min(times)
            rebal.append({"config": f"configs[{idx}] genz {fid} d={d} rtol={tau:g}, {per * world} initial subdomains, "
                                    f"first {its} iterations", "seconds_wall_max_over_ranks": t,
                          "evals": drx.result.total_f_evals, "evals_per_s": drx.result.total_f_evals / t,
                          "messages": drx.messages_total, "regions_transferred": drx.regions_transferred_total,
                          "peak_regions": drx.result.peak_regions, "integral": drx.result.integral,
                          "error": drx.result.error, "termination_reason": drx.result.termination_reason.value,
                          "per_rank_idle_s": [round(x.idle_seconds, 4) for x in drx.timings]})
        dr0 = res[0][0]
        evals = sum(r[0].result.total_f_evals for r in res)
        if rank != 0:
            return None
        peak_tf, peak_src = peak()
        return {
            "metric": "integrand_evals_per_s", "value": evals / t_dev, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"genz_f2_product_peak_d8_rtol1e-6_init64_fixed{args.iterations}its",
                "integrand": "f2 (Genz product peak, a=50^-2)", "d": D, "rtol": TAU, "initial_regions": INIT,
                "iterations": args.iterations, "evals_per_step": dr0.result.total_f_evals,
                "peak_regions": dr0.result.peak_regions, "messages_per_step": dr0.messages_total,
                "regions_transferred_per_step": dr0.regions_transferred_total,
                "termination_reason": dr0.result.termination_reason.value,
                "parallelism": f"round-robin redistribution over {world} ranks ({backend})",
                "l2": "late-iteration stores exceed L2",
            },
            "roofline": {"bound": "fp64", "kernel": "k1_gm_eval", "peak": peak_tf * world, "unit": "TFLOP/s",
                         "achieved": evals * F_FLOPS / t_dev / 1e12,
                         "frac": evals * F_FLOPS / t_dev / 1e12 / (peak_tf * world),
                         "traffic": traffic[0] if traffic else None,
                         "traffic_detail": traffic[1] if traffic else None,
                         "peak_source": peak_src + f" x {world} GPUs", "flops_per_eval": F_FLOPS},
            # per iteration and rank: the evaluate and classify status reads (2 x 144 B)
            "e2e": {"value": evals / t_wall, "unit": "evals/s", "h2d_bytes_per_step": 2 * INIT * D * 8,
                    "d2h_bytes_per_step": 2 * 144 * args.iterations * world},
            "gpu_launches": sum((r[0].device_stats or {}).get("launches", 0) for r in res),
            "clocks": clk.summary(),
            "time_to_tolerance": [{
                "config": "configs[1] genz f2 d=5 rtol=1e-06, run_distributed, 8 initial subdomains per rank",
                "seconds_wall_max_over_ranks": ttt[len(ttt) // 2], "termination_reason":
                dr5.result.termination_reason.value, "iterations": dr5.result.iterations,
                "integral": dr5.result.integral, "error": dr5.result.error, "evals": dr5.result.total_f_evals,
                "peak_regions": dr5.result.peak_regions, "messages": dr5.messages_total,
                "regions_transferred": dr5.regions_transferred_total}],
            "rebalancing": rebal,
        }
    finally:
        dist.destroy_process_group()
