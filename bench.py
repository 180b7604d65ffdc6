#!/usr/bin/env python
"""Benchmark: integrand evaluations/s of the B200 adaptive-cubature hot path.

Workload (BASELINE.json north star, configs[2]): Genz product peak f2,
d = 8, rtol 1e-6.  The reference algorithm can never reach that tolerance
(the finalized-error carry exceeds the budget), so the
step is the survey's fixed-work definition (sec.8d): `integrate` from a fixed
64-subdomain partition for exactly N_it iterations - identical region sets
for every GPU count, K1 -> K2 -> K3 each iteration, regions resident in HBM.

  python bench.py [--gpus N --steps K --warmup W --iterations N_it]
  python bench.py --impl reference ...   # the reference algorithm on host cores

value      = total integrand evaluations / device time (CUDA events on the
             library's stream around the whole loop), summed over K steps
e2e        = same evaluations / wall time of the public `integrate()` call
             (host partition -> device, per-iteration status -> host)
roofline   = kernel K1 (k1_gm_eval): algorithmic FP64 flops F(d)=6d+5 per
             evaluation / K1 event time, vs the measured FP64
             peak of this B200 (tools/fp64_peak, DFMA throughput)
N > 1      = torchrun, one rank per GPU; the 64 subdomains are dealt
             round-robin (ref distributed.py:371-378), ranks run the
             redistribution protocol; max over ranks of the device time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D = 8
FN = "f2"
TAU = 1e-6
INIT = 64
F_FLOPS = 6 * D + 5  # algorithmic FP64 flops per evaluation (f2)
DEFAULT_ITERS = 26  # largest fixed-work step whose store fits one B200 (249 M regions)
CPU_SAMPLE_ITERS = 11  # oracle: ~50.6 M evaluations, ~10 s on one host core
REF_STEP_ITERS = 12    # reference arm: ~93 M evaluations per step


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak_tflops():
    """Measured FP64 peak (DFMA throughput), live if the probe is built."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
            return json.loads(out)["fp64_tflops"], "measured live (tools/fp64_peak: DFMA, all SMs)"
        except Exception:
            pass
    with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as fh:
        return json.load(fh)["fp64_tflops"], "measured r01 (profiles/r01_fp64_peak.json)"


def ncu_traffic():
    """(dram bytes read + written per K1 launch, detail) from the committed
    ncu --set full summary of one large K1 launch (profiles/k1_ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "k1_ncu_summary.json")
    if os.path.exists(p):
        with open(p) as fh:
            s = json.load(fh)
        return s["dram_bytes_per_launch"], {
            "regions_in_launch": s["regions_in_launch"], "bytes_per_region": s["dram_bytes_per_region"],
            "algorithmic_bytes_per_region": s["algorithmic_bytes_per_region"],
            "fp64_pipe_active_pct": s["fp64_pipe_active_pct"],
            "fp64_instructions_per_eval": s["fp64_instructions_per_eval"],
            "source": "profiles/k1_ncu_summary.json"}
    return None, None


REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # offline install of the unmodified reference (travels to the box)


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity_cores": aff,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS")}


def reference_package():
    """The reference's own `hcub` (pip-installed into baseline/_ref), or None."""
    if not os.path.isfile(os.path.join(REF_DIR, "hcub", "driver.py")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import hcub
    return hcub


def cpu_baseline():
    """The reference's own `integrate` (single process) on a bounded sample
    of the workload; the numpy port (oracle/) if the reference is absent."""
    ref = reference_package()
    t0 = time.perf_counter()
    if ref is not None:
        r = ref.integrate(ref.make_integrand(FN, D).evaluate, ref.HyperRect.unit_cube(D),
                          ref.DriverConfig(TAU, max_iterations=CPU_SAMPLE_ITERS, max_regions=1 << 40),
                          initial_regions=INIT)
        kind, what = "reference", "reference hcub.integrate (baseline/_ref, unmodified)"
    else:
        from oracle import hcub_oracle as orc
        r = orc.integrate(orc.integrand(FN, D), D, TAU, init=INIT, max_iterations=CPU_SAMPLE_ITERS)
        kind, what = "port", "oracle integrate (numpy restatement of the reference)"
    dt = time.perf_counter() - t0
    return {"value": r.total_f_evals / dt, "unit": "evals/s", "cores": 1, "kind": kind,
            "sample": f"{what}(f2, d=8, rtol 1e-6, init=64), first {CPU_SAMPLE_ITERS} iterations = "
                      f"{r.total_f_evals} evaluations in {dt:.2f} s (one process)", "host": host_info()}


def run_reference(args, rank, world):
    """The reference's own multi-worker CPU path on the host cores:
    `run_distributed(backend="concurrent", workers=P)` of the unmodified
    reference (one thread per worker, ref distributed.py:659-848) with
    64/P initial subdomains per rank - the same region set as the GPU
    workload - each step a bounded prefix of it.  P is the faster of 8 and
    the largest power of two <= the host cores, chosen in the warm-up.
    Falls back to the numpy port over a process pool without the package."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    ref = reference_package()
    if ref is not None:
        f = ref.make_integrand(FN, D).evaluate
        cfg = ref.DriverConfig(TAU, max_iterations=REF_STEP_ITERS, max_regions=1 << 40)
        pmax = 1
        while pmax * 2 <= min(cores, INIT):
            pmax *= 2
        cands = sorted({min(8, pmax), pmax})

        def once(P):
            t0 = time.perf_counter()
            dr = ref.run_distributed(f, ref.HyperRect.unit_cube(D), cfg,
                                     ref.RedistributionConfig(initial_subdomains_per_rank=INIT // P), workers=P,
                                     backend="concurrent")
            return dr.result.total_f_evals, time.perf_counter() - t0

        rates = {}
        for s in range(max(args.warmup, len(cands))):
            P = cands[s % len(cands)]
            ev, dt = once(P)
            rates[P] = max(rates.get(P, 0.0), ev / dt)
        P = max(rates, key=rates.get)
        kind = "reference"
        sample = (f"reference hcub.run_distributed(backend='concurrent', workers={P}) from baseline/_ref "
                  f"(unmodified), {INIT // P} initial subdomains per rank, first {REF_STEP_ITERS} iterations "
                  f"per step; warm-up rates by workers: " + ", ".join(f"{k}: {v:.3g}" for k, v in sorted(rates.items())))
        threads = P
    else:
        from oracle import hcub_oracle as orc

        def once(_):
            t0 = time.perf_counter()
            ev, _ = orc.integrate_parallel(FN, D, TAU, INIT, REF_STEP_ITERS, cores)
            return ev, time.perf_counter() - t0

        for _ in range(args.warmup):
            once(None)
        P, kind, threads = None, "port", cores
        sample = f"numpy port (oracle/), first {REF_STEP_ITERS} iterations per step over a {cores}-process pool"
    times, evals = [], 0
    for _ in range(args.steps):
        ev, dt = once(P)
        times.append(dt)
        evals += ev
    v = evals / sum(times)
    line = {
        "impl": "reference", "metric": "integrand_evals_per_s", "value": v, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"genz_f2_product_peak_d8_rtol1e-6_init64_first{REF_STEP_ITERS}its",
                   "note": "the reference's own CPU path on all host cores; a bounded prefix of the same "
                           "fixed-work workload (the full 26 iterations are ~2.4e11 evaluations, hours on CPU)"},
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": threads, "kind": kind, "sample": sample,
                         "host": host_info()},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


TTT_CONFIGS = [
    # (BASELINE configs[] index, integrand, d, rtol, initial regions, repetitions, reference CPU behaviour[, rule])
    (0, "f4", 3, 1e-6, None, 5, "tolerance at iteration 17 after 0.054 s (SURVEY.md 8d)"),
    (1, "f2", 5, 1e-6, None, 5, "max_regions (2^24) at iteration 28 after 585 s, not converged (SURVEY.md 8d)"),
    # the paper's "9-order" rule (rule9.py, generator kernel k1_gm9_eval) on the same config
    (1, "f2", 5, 1e-6, None, 5, "degree-7 reference: max_regions (2^24) at iteration 28 after 585 s", "gm9"),
    (3, "f3", 10, 1e-5, 80, 1, "iteration 28 after 2,673 s, eps 4.1e-15 > floor 1e-16, not converged (SURVEY.md 8d)"),
    (3, "f3", 10, 1e-5, 80, 3, "degree-7 reference: eps 4.1e-15 > floor 1e-16 after 2,673 s", "gm9"),
    # infeasible under the reference algorithm: runs until the store fills HBM
    (4, "f6", 6, 1e-4, 48, 3, "max_regions (2^24) at iteration 25 after 733 s, eps/I 0.029, true error 39 % "
                              "(SURVEY.md 8d)"),
]


def time_to_tolerance(hb, torch, dev):
    """BASELINE configs[0], [1], [3] and [4] run to the reference's own
    stopping rule on one B200 with max_regions sized to HBM (the CPU
    reference stops at its 2^24-region guard / is far from converged; [4]
    cannot converge and ends when the store fills HBM).  Median over
    repetitions of the device time; one untimed warm run first."""
    out = []
    for idx, fid, d, tau, init, reps, ref, *rule in TTT_CONFIGS:
        rule = rule[0] if rule else "gm"
        f = hb.make_integrand(fid, d)
        cfg = hb.DriverConfig(tau, max_regions=1 << 40, rule=rule)
        runs = []
        for i in range(reps + 1):
            st = {}
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            r = hb.integrate(f, hb.HyperRect.unit_cube(d), cfg, initial_regions=init, stats=st)
            wall = time.perf_counter() - t0
            if i:
                runs.append((st["device_ms"] * 1e-3, wall, r))
        runs.sort(key=lambda x: x[0])
        t_dev, wall, r = runs[len(runs) // 2]
        exact = f.reference_value
        out.append({"config": f"configs[{idx}] genz {fid} d={d} rtol={tau:g}" + (f" init={init}" if init else "")
                    + (f" rule={rule}" if rule != "gm" else ""),
                    "seconds_device": t_dev, "seconds_wall": wall,
                    "termination_reason": r.termination_reason.value, "iterations": r.iterations,
                    "integral": r.integral, "error": r.error, "true_rel_error": abs(r.integral - exact) / abs(exact),
                    "evals": r.total_f_evals, "peak_regions": r.peak_regions, "evals_per_s": r.total_f_evals / t_dev,
                    "error_over_integral": r.error / abs(r.integral) if r.integral else None,
                    # ref driver.py:174-175: eps <= max(abs_floor, |I| * rtol) - which term governed the stop,
                    # and whether the north star's "achieved relative error <= rtol" holds
                    "stopping_budget": max(cfg.abs_floor, abs(r.integral) * tau),
                    "stopping_rule_governed_by": "abs_floor" if cfg.abs_floor > abs(r.integral) * tau else "rtol",
                    "true_rel_error_le_rtol": abs(r.integral - exact) / abs(exact) <= tau,
                    "reference_cpu": ref})
    return out


def flush_l2(torch, dev):
    buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    torch.cuda.synchronize(dev)


def run_single(args):
    import torch

    import paper_2511_01573_b200 as hb

    dev = 0
    torch.cuda.set_device(dev)
    hb.set_device(dev)
    f = hb.make_integrand(FN, D)
    dom = hb.HyperRect.unit_cube(D)
    cfg = hb.DriverConfig(TAU, max_iterations=args.iterations, max_regions=1 << 40)
    peak_tf, peak_src = fp64_peak_tflops()

    def step():
        st = {}
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        r = hb.integrate(f, dom, cfg, initial_regions=INIT, stats=st)
        wall = time.perf_counter() - t0
        return r, st, wall

    for _ in range(args.warmup):
        step()
        flush_l2(torch, dev)
    res = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            res.append(step())
            flush_l2(torch, dev)
    torch.cuda.synchronize(dev)
    evals = sum(r.total_f_evals for r, _, _ in res)
    dev_s = sum(st["device_ms"] for _, st, _ in res) * 1e-3
    wall_s = sum(w for _, _, w in res)
    k1_s = sum(st["k1_ms"] for _, st, _ in res) * 1e-3
    k1_launches = sum(st["k1_launches"] for _, st, _ in res)
    launches = sum(st["launches"] for _, st, _ in res)
    r0, st0, _ = res[0]
    achieved_tf = evals * F_FLOPS / k1_s / 1e12
    traffic, traffic_detail = ncu_traffic()
    h2d = 2 * INIT * D * 8 + 2 * D * 8
    d2h = args.iterations * 144
    line = {
        "metric": "integrand_evals_per_s", "value": evals / dev_s, "unit": "evals/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": f"genz_f2_product_peak_d8_rtol1e-6_init64_fixed{args.iterations}its",
            "integrand": "f2 (Genz product peak, a=50^-2)", "d": D, "rtol": TAU, "initial_regions": INIT,
            "iterations": args.iterations, "evals_per_step": r0.total_f_evals, "peak_regions": r0.peak_regions,
            "termination_reason": r0.termination_reason.value, "integral": r0.integral, "error": r0.error,
            "l2": "flushed between steps (512 MiB device write); late-iteration stores exceed L2",
            "parallelism": "single device",
        },
        "roofline": {
            # neither HBM nor tensor cores: K1 is bound by the FP64 vector pipe (no dense
            # contraction to map onto tcgen05); peak = measured DFMA rate
            "bound": "fp64", "kernel": "k1_gm_eval", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": achieved_tf / peak_tf, "traffic": traffic, "traffic_detail": traffic_detail,
            "peak_source": peak_src,
            "flops_per_eval": F_FLOPS, "k1_evals_per_s": evals / k1_s,
            "k1_share_of_step": k1_s / dev_s,
            # executed FP64 instructions (ncu, incl. the exact-path nodes) issued per second
            # against the measured DFMA instruction rate (peak / 2 flops)
            "fp64_instruction_issue_frac": (evals / k1_s * traffic_detail["fp64_instructions_per_eval"]
                                            / (peak_tf * 1e12 / 2)) if traffic_detail else None,
        },
        "e2e": {"value": evals / wall_s, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "k1_launches": k1_launches,
        "clocks": clk.summary(),
    }
    line["time_to_tolerance"] = time_to_tolerance(hb, torch, dev)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)


def run_multi(args, rank, world):
    from paper_2511_01573_b200.bench_dist import run_multi_gpu
    line = run_multi_gpu(args, rank, world, D=D, FN=FN, TAU=TAU, INIT=INIT, F_FLOPS=F_FLOPS,
                         peak=fp64_peak_tflops, clock_sampler=ClockSampler, traffic=ncu_traffic())
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iterations", type=int, default=DEFAULT_ITERS)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        return run_multi(args, rank, world)
    return run_single(args)


if __name__ == "__main__":
    main()
