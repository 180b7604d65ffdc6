"""One time-to-tolerance run (BASELINE configs[1] by default) for ncu launch lists:
  python tools/profile_ttt.py [fn d tau init]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb

fn = sys.argv[1] if len(sys.argv) > 1 else "f2"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 5
tau = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
init = int(sys.argv[4]) if len(sys.argv) > 4 else None
st = {}
r = hb.integrate(hb.make_integrand(fn, d), hb.HyperRect.unit_cube(d), hb.DriverConfig(tau, max_regions=1 << 40),
                 initial_regions=init, stats=st)
print(r, st)
