"""Per-iteration region counts / device time of the bench workload."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb
maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 26
tr = []
st = {}
t = time.time()
r = hb.integrate(hb.make_integrand("f2", 8), hb.HyperRect.unit_cube(8), hb.DriverConfig(1e-6, max_iterations=maxit, max_regions=1 << 40),
                 trace=tr.append, initial_regions=64, stats=st)
w = time.time() - t
print(json.dumps(dict(result=str(r), wall=w, stats=st, trace=[[x.iteration, x.active_regions, x.integral, x.error, x.f_evals] for x in tr])))
