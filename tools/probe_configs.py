"""Per-iteration wall times of the bench workload and the other BASELINE
configs on one B200 (max_regions sized to HBM)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb


def run(name, fid, d, tau, maxit, init=None, max_regions=1 << 40):
    f = hb.make_integrand(fid, d)
    stamps = []
    t0 = time.perf_counter()
    tr = []
    def cb(t):
        stamps.append(time.perf_counter() - t0)
        tr.append(t)
    st = {}
    r = hb.integrate(f, hb.HyperRect.unit_cube(d), hb.DriverConfig(tau, max_iterations=maxit, max_regions=max_regions),
                     trace=cb, initial_regions=init, stats=st)
    w = time.perf_counter() - t0
    exact = f.reference_value
    print(json.dumps(dict(case=name, reason=r.termination_reason.value, iterations=r.iterations, integral=r.integral,
                          error=r.error, rel_err_true=abs(r.integral - exact) / abs(exact), eps_over_I=r.error / abs(r.integral),
                          evals=r.total_f_evals, peak=r.peak_regions, wall_s=w, stats=st,
                          per_iter=[[t.iteration, t.active_regions, round(s * 1e3, 3)] for t, s in zip(tr, stamps)])), flush=True)


which = sys.argv[1:] or ["bench", "d5", "f3", "f6", "f4"]
if "bench" in which:
    run("f2_d8_init64_26its", "f2", 8, 1e-6, 26, init=64)
if "d5" in which:
    run("f2_d5_t2t", "f2", 5, 1e-6, 1000)
if "f4" in which:
    run("f4_d3_t2t", "f4", 3, 1e-6, 1000)
if "f3" in which:
    run("f3_d10_32its", "f3", 10, 1e-5, 32, init=80)
if "f6" in which:
    run("f6_d6_30its", "f6", 6, 1e-4, 30, init=48)
