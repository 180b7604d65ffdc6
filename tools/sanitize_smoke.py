"""Small end-to-end exercise of every kernel family for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_01573_b200 as hb
from paper_2511_01573_b200.rules import parse_rule_table

f = hb.make_integrand("f2", 5)
r = hb.integrate(f, hb.HyperRect.unit_cube(5), hb.DriverConfig(1e-4, max_iterations=9))
print("integrate", r.termination_reason.value, r.iterations)
hb.set_k1_lanes(0)  # one-region-per-lane kernel (phase barriers, fused sums) on a small store
r = hb.integrate(f, hb.HyperRect.unit_cube(5), hb.DriverConfig(1e-4, max_iterations=7))
hb.set_k1_lanes(-1)
print("integrate lane1", r.termination_reason.value, r.iterations)
pp = hb.make_product_peak(4, center=0.1)[0]
dr = hb.run_distributed(pp, hb.HyperRect.unit_cube(4), hb.DriverConfig(1e-4, max_iterations=12), workers=3,
                        collect_log=True)
print("distributed", dr.messages_total, dr.regions_transferred_total, dr.result.iterations)
t = hb.build_gm_rule(3)
txt = "\n".join(" ".join(map(repr, list(o.generator) + [o.weight, o.embedded_weight])) for o in t.orbits)
lo = np.random.default_rng(0).random((300, 3)) * 0.5
hi = lo + 0.25
print("table", hb.apply_rule_batch(parse_rule_table(txt), lo, hi, hb.make_integrand("f4", 3))[3])
print("gk", hb.apply_rule_batch(hb.build_gk_tensor_rule(3), lo, hi, hb.make_integrand("f4", 3))[3])
r1 = hb.integrate(hb.make_integrand("f2", 1), hb.HyperRect.unit_cube(1), hb.DriverConfig(1e-8))
print("d1", r1.termination_reason.value)
from paper_2511_01573_b200.driver import device_exact_sum
print("fsum", device_exact_sum(np.random.default_rng(1).standard_normal(10000)))
# overlapped evaluation: K1 on the store, rows appended meanwhile, tail K1 into the same sums
from paper_2511_01573_b200.regions import partition_arrays
from paper_2511_01573_b200.worker import DeviceWorker
w = DeviceWorker(hb.build_gm_rule(4), hb.make_integrand("f2", 4), hb.HyperRect.unit_cube(4))
lo, hi = partition_arrays(hb.HyperRect.unit_cube(4), 16)
w.append(lo, hi)
I, E, _ = w.evaluate()
w.classify(I, hb.DriverConfig(1e-6))
w.evaluate_begin()
w.append(lo[:5] * 0.5, hi[:5] * 0.5)
print("overlap", w.evaluate_end())
w.close()
# degree-9 rule: node-table kernel with lane groups (small store), then the
# generator kernel k1_gm9_eval once the store exceeds 128 regions per SM
r9 = hb.integrate(f, hb.HyperRect.unit_cube(5), hb.DriverConfig(1e-7, max_iterations=14, rule="gm9"))
print("gm9", r9.termination_reason.value, r9.iterations, r9.peak_regions)
# take_top on virtual children (donor side), removed children skipped by the next K1
dr = hb.run_distributed(pp, hb.HyperRect.unit_cube(4), hb.DriverConfig(1e-6, max_iterations=10),
                        hb.RedistributionConfig(cap=16, initial_subdomains_per_rank=2), workers=4,
                        backend="concurrent", collect_log=True)
print("distributed cap16", dr.messages_total, dr.regions_transferred_total, dr.result.iterations)
