"""One f2 d=8 fixed-work integration (init 64) for ncu captures:
  python tools/profile_k1.py <iterations>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01573_b200 as hb

it = int(sys.argv[1]) if len(sys.argv) > 1 else 20
fn = sys.argv[2] if len(sys.argv) > 2 else "f2"
d = int(sys.argv[3]) if len(sys.argv) > 3 else 8
st = {}
r = hb.integrate(hb.make_integrand(fn, d), hb.HyperRect.unit_cube(d), hb.DriverConfig(1e-6, max_iterations=it, max_regions=1 << 40),
                 initial_regions=64, stats=st)
print(r, st)
