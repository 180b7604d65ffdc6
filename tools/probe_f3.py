import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb
d = 10
f = hb.make_integrand("f3", d)
for maxit in (40,):
    tr = []
    st = {}
    t0 = time.perf_counter()
    r = hb.integrate(f, hb.HyperRect.unit_cube(d), hb.DriverConfig(1e-5, max_iterations=maxit, max_regions=1 << 40),
                     trace=tr.append, initial_regions=80, stats=st)
    w = time.perf_counter() - t0
    print(json.dumps(dict(reason=r.termination_reason.value, it=r.iterations, I=r.integral, E=r.error,
                          target=max(1e-16, abs(r.integral) * 1e-5), true_rel=abs(r.integral - f.reference_value) / f.reference_value,
                          evals=r.total_f_evals, peak=r.peak_regions, wall=w, stats=st,
                          tail=[[t.iteration, t.active_regions, t.error] for t in tr[-8:]])))
