"""Drive the HBM-bound store kernels at scale for ncu: the fused-split
integrate loop (k2_reduce, k3_classify, k_scan_tiles, k3_compact) and one
worker-mode iteration with explicit materialisation (k3_split, k3_expand,
k4 take-top, k_keep_*).  usage: python tools/profile_store.py <iterations>"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200 import _lib
from paper_2511_01573_b200.regions import partition_arrays
from paper_2511_01573_b200.worker import DeviceWorker

its = int(sys.argv[1]) if len(sys.argv) > 1 else 22
d = 8
f = hb.make_integrand("f2", d)
dom = hb.HyperRect.unit_cube(d)
cfg = hb.DriverConfig(1e-6, max_iterations=its, max_regions=1 << 40)
hb.integrate(f, dom, cfg, initial_regions=64)
# worker mode: explicit split (split=1), then expand via a virtual split + take_top
w = DeviceWorker(hb.build_gm_rule(d), f, dom)
lo, hi = partition_arrays(dom, 64)
w.append(lo, hi)
cd = cfg.descriptor()
for it in range(its - 2):
    I, E, _ = w.evaluate()
    out = _lib.hcub_classify_out()
    mode = 1 if it == its - 3 else 2  # last one: explicit K3 split
    _lib.check(_lib.lib().hcub_worker_classify(w._h, I, C.byref(cd), mode, C.byref(out)))
I, E, _ = w.evaluate()
w.classify(I, cfg)          # virtual children
w.take_top(512)             # -> k3_expand + K4 + removal
print("regions", len(w))
w.close()
