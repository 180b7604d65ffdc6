"""run_distributed on device workers (B200) vs the reference's own
deterministic_sim logs: identical region flow (counts, transfers, census,
virtual time columns), estimates to 1e-12 relative.  Plus a two-process
process-group run on one GPU (host-tensor transport) and take_top/append
round trips on the device store."""
import math
import os
import socket

import numpy as np
import pytest

from conftest import domain_of, golden_names, load_json

import paper_2511_01573_b200 as hb

pytestmark = pytest.mark.gpu


def run_case(name, workers=None, backend="deterministic_sim"):
    g = load_json("dist", name)
    spec = g["spec"]
    dlo, dhi = domain_of(spec)
    if spec["f"] == "pp":
        f = hb.make_product_peak(spec["d"], spec.get("center", 0.5), spec.get("sharpness", 50.0))[0]
    else:
        f = hb.make_integrand(spec["f"], spec["d"])
    rcfg = hb.RedistributionConfig(cap=spec.get("cap", 512), initial_subdomains_per_rank=spec.get("per_rank", 8),
                                   delivery_latency=spec.get("latency", 1))
    dr = hb.run_distributed(f, hb.HyperRect(dlo, dhi), hb.DriverConfig(spec["tau"]), rcfg,
                            workers=workers or spec["P"], backend=backend, collect_log=True)
    return g, dr


def _strict(name):
    # libm/BLAS integrands (f3: pow, f6: exp) may flip a rounding-decided axis late
    return not name.startswith(("f3", "f6"))


@pytest.mark.parametrize("backend", ["deterministic_sim", "concurrent"])
@pytest.mark.parametrize("name", golden_names("dist"))
def test_device_engine_matches_reference(name, backend):
    """Device workers vs the reference's logs.  "concurrent" runs one thread
    per rank through the process-group code path (`_TorchTransport`) with
    device tensors: K4 gathers the donor's rows into a CUDA tensor, the
    transfer is an event-ordered device copy left in flight across the next
    K1, K5 appends from the device buffer - the NCCL data path on one GPU."""
    from paper_2511_01573_b200 import distributed as D
    from paper_2511_01573_b200.worker import DeviceWorker
    used = {"take_top_device": 0, "append_device": 0, "evaluate_begin": 0}
    wrapped = {}
    if backend == "concurrent":
        for nm in used:
            fn = getattr(DeviceWorker, nm)
            wrapped[nm] = fn

            def w(self, *a, _fn=fn, _nm=nm, **k):
                used[_nm] += 1
                return _fn(self, *a, **k)
            setattr(DeviceWorker, nm, w)
    try:
        g, dr = run_case(name, backend=backend)
    finally:
        for nm, fn in wrapped.items():
            setattr(DeviceWorker, nm, fn)
    if backend == "concurrent" and g["messages_total"]:
        assert used["take_top_device"] > 0 and used["append_device"] > 0 and used["evaluate_begin"] > 0
    if not _strict(name):
        res = g["result"]
        assert dr.result.termination_reason.value == res["termination_reason"]
        assert abs(dr.result.iterations - res["iterations"]) <= 1
        assert math.isclose(dr.result.integral, res["integral"], rel_tol=1e-6)
        return
    res = g["result"]
    assert dr.result.termination_reason.value == res["termination_reason"]
    assert dr.result.iterations == res["iterations"]
    assert dr.result.total_f_evals == res["total_f_evals"]
    assert dr.result.peak_regions == res["peak_regions"]
    assert math.isclose(dr.result.integral, res["integral"], rel_tol=1e-12)
    assert math.isclose(dr.result.error, res["error"], rel_tol=1e-9)
    assert dr.messages_total == g["messages_total"]
    assert dr.regions_transferred_total == g["regions_transferred_total"]
    for mine, ref in zip(dr.iteration_log, g["log"]):
        for key in ("counts", "post_split_counts", "inflight_regions", "inflight_batches", "census"):
            assert mine[key] == ref[key], (key, mine["iteration"])
        assert [list(t) for t in mine["transfers"]] == [list(t) for t in ref["transfers"]]
        assert math.isclose(mine["global_integral"], ref["global_integral"], rel_tol=1e-12)
    for t, rt in zip(dr.timings, g["timings"]):
        assert (t.messages_out, t.regions_out) == (rt["messages_out"], rt["regions_out"])
        if backend == "deterministic_sim":  # virtual time columns (ref :506-510)
            assert (t.compute_seconds, t.idle_seconds) == (rt["compute"], rt["idle"])


def test_concurrent_backend_same_numerics():
    g, dr = run_case("pp_d4_c01_P4", backend="concurrent")
    assert dr.result.iterations == g["result"]["iterations"]
    assert math.isclose(dr.result.integral, g["result"]["integral"], rel_tol=1e-12)
    assert all(t.compute_seconds > 0 for t in dr.timings)


def test_take_top_matches_numpy_stable_argsort():
    """K4 selection order == np.argsort(-error, kind='stable') with heavy ties."""
    from paper_2511_01573_b200.worker import DeviceWorker
    d = 3
    table = hb.build_gm_rule(d)
    f = hb.make_integrand("f4", d)
    w = DeviceWorker(table, f, hb.HyperRect.unit_cube(d))
    rng = np.random.default_rng(5)
    n = 5000
    lo = rng.random((n, d)) * 0.5
    hi = lo + 0.25 + rng.random((n, d)) * 0.1
    err = np.round(rng.random(n) * 20) / 4  # many exact ties
    err[::97] = 0.0
    integ = rng.standard_normal(n)
    w.append(lo, hi, integ, err)
    for take in (1, 7, 512, 600):
        order = np.argsort(-err, kind="stable")[:take]
        tl, th, te, ti = w.take_top(take)
        assert np.array_equal(tl, lo[order]) and np.array_equal(th, hi[order])
        assert np.array_equal(te, err[order]) and np.array_equal(ti, integ[order])
        keep = np.ones(len(err), dtype=bool)
        keep[order] = False
        lo, hi, err, integ = lo[keep], hi[keep], err[keep], integ[keep]
        rlo, rhi, rI, rE, _ = w.read()
        assert np.array_equal(rlo, lo) and np.array_equal(rE, err) and np.array_equal(rI, integ)
    w.close()


def _grown_worker(d, fid, its):
    """A device worker after `its` evaluate/classify rounds of the protocol
    (post-split store with virtual children)."""
    from paper_2511_01573_b200.regions import partition_arrays
    from paper_2511_01573_b200.worker import DeviceWorker
    dom = hb.HyperRect.unit_cube(d)
    w = DeviceWorker(hb.build_gm_rule(d), hb.make_integrand(fid, d), dom)
    lo, hi = partition_arrays(dom, 16)
    w.append(lo, hi)
    cfg = hb.DriverConfig(1e-9)
    for _ in range(its):
        I, _, _ = w.evaluate()
        w.classify(I, cfg)
    return w


@pytest.mark.parametrize("fid,d,its", [("f2", 3, 7), ("f4", 4, 8), ("f6", 3, 6)])
def test_take_top_on_virtual_children_equals_materialized(fid, d, its):
    """take_top right after classify selects over the survivors' columns and
    leaves the removed children to the next K1 (no expansion, no store
    rewrite); batch, remaining store and the next evaluation equal the
    general path on the materialised children = np.argsort(-E, 'stable')
    over the post-split store (ref distributed.py:381-392)."""
    for take in (1, 2, 7, 64, 511, 512):
        a, b = _grown_worker(d, fid, its), _grown_worker(d, fid, its)
        try:
            blo, bhi, bI, bE, _ = b.read()  # materialises b's children: the general path
            take = min(take, len(bE))
            order = np.argsort(-bE, kind="stable")[:take]
            ta = a.take_top(take)
            tb = b.take_top(take)
            for x, y in zip(ta, tb):
                assert np.array_equal(x, y)
            assert np.array_equal(ta[0], blo[order]) and np.array_equal(ta[2], bE[order])
            assert len(a) == len(b) == len(bE) - take
            ra, rb = a.evaluate(), b.evaluate()
            assert ra == rb
            for x, y in zip(a.read(), b.read()):
                assert np.array_equal(x, y)
        finally:
            a.close()
            b.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hb.set_device(0)
        g, dr = run_case("pp_d4_c01_P2", workers=2, backend="nccl")
        out.put((rank, dr.result.integral, dr.result.iterations, dr.result.total_f_evals, dr.messages_total,
                 [(e["counts"], e["transfers"]) for e in dr.iteration_log]))
    finally:
        dist.destroy_process_group()


def test_process_group_two_ranks_one_gpu():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    g = load_json("dist", "pp_d4_c01_P2")
    for o in outs:
        assert o[2] == g["result"]["iterations"] and o[3] == g["result"]["total_f_evals"]
        assert math.isclose(o[1], g["result"]["integral"], rel_tol=1e-12)
        assert o[4] == g["messages_total"]
        assert [(c, [list(t) for t in tr]) for c, tr in o[5]] == \
               [(e["counts"], [list(t) for t in e["transfers"]]) for e in g["log"]]


def _nccl_single(port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        from paper_2511_01573_b200.worker import DeviceWorker
        used = {"exchange_records": 0, "classify_commit": 0, "classify": 0}
        for nm in used:
            fn = getattr(DeviceWorker, nm)

            def w(self, *a, _fn=fn, _nm=nm, **k):
                used[_nm] += 1
                return _fn(self, *a, **k)
            setattr(DeviceWorker, nm, w)
        hb.set_device(0)
        g, dr = run_case("pp_d4_c01_P2", workers=1, backend="nccl")
        # a run stopped by the iteration cap: its last iteration launches no classify
        f = hb.make_integrand("f2", 5)
        capped = hb.run_distributed(f, hb.HyperRect.unit_cube(5), hb.DriverConfig(1e-9, max_iterations=7),
                                    workers=1, backend="nccl")
        out.put((dr.result.integral, dr.result.error, dr.result.iterations, dr.result.total_f_evals,
                 [e["counts"] for e in dr.iteration_log],
                 [(e["global_integral"], e["global_error"]) for e in dr.iteration_log], used,
                 (capped.result.integral, capped.result.error, capped.result.iterations,
                  capped.result.termination_reason.value)))
    finally:
        dist.destroy_process_group()


def test_nccl_transport_single_rank_matches_in_process():
    """The NCCL transport on a one-rank group - the one-sync protocol: record
    rows all-gathered over the native communicator (hcub_comm_init /
    hcub_worker_exchange_records), global integral reduced on the device,
    classify launched speculatively and committed - gives exactly the
    in-process result, iteration by iteration."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_single, args=(_free_port(), q))
    p.start()
    got = q.get(timeout=600)
    p.join(timeout=60)
    g, dr = run_case("pp_d4_c01_P2", workers=1)
    assert got[0] == dr.result.integral and got[1] == dr.result.error
    assert got[2] == dr.result.iterations and got[3] == dr.result.total_f_evals
    assert got[4] == [e["counts"] for e in dr.iteration_log]
    assert got[5] == [(e["global_integral"], e["global_error"]) for e in dr.iteration_log]
    used = got[6]
    assert used["exchange_records"] >= dr.result.iterations  # every record exchange went native
    assert used["classify"] == 0
    ref = hb.run_distributed(hb.make_integrand("f2", 5), hb.HyperRect.unit_cube(5),
                             hb.DriverConfig(1e-9, max_iterations=7), workers=1)
    assert got[7] == (ref.result.integral, ref.result.error, ref.result.iterations, "max_iterations")


@pytest.mark.parametrize("lanes", [-1, 0])
def test_evaluate_begin_end_equals_deliver_then_evaluate(lanes):
    """The overlapped order (K1 on the store, rows appended meanwhile, a tail
    K1 into the same exact accumulators) gives the same rows, estimates and
    bit-identical exact partials as appending first and evaluating after -
    both right after a split (virtual children, fused-split K1) and on a
    plain row store."""
    from paper_2511_01573_b200.regions import partition_arrays
    from paper_2511_01573_b200.worker import DeviceWorker
    d = 5
    f = hb.make_integrand("f2", d)
    dom = hb.HyperRect.unit_cube(d)
    cfg = hb.DriverConfig(1e-6)
    lo, hi = partition_arrays(dom, 40)
    rng = np.random.default_rng(7)
    alo = rng.random((300, d)) * 0.5
    ahi = alo + rng.random((300, d)) * 0.5 + 1e-3
    hb.set_k1_lanes(lanes)
    try:
        outs = []
        for overlapped in (False, True):
            w = DeviceWorker(hb.build_gm_rule(d), f, dom)
            w.append(lo, hi)
            I, E, _ = w.evaluate()
            w.classify(I, cfg)  # children now virtual
            for rnd in range(2):
                if overlapped:
                    w.evaluate_begin()
                    w.append(alo[rnd::2], ahi[rnd::2])
                    got = w.evaluate_end()
                else:
                    w.append(alo[rnd::2], ahi[rnd::2])
                    got = w.evaluate()
                outs.append((overlapped, rnd, got, w.read()))
                w.classify(got[0], cfg)
            w.close()
    finally:
        hb.set_k1_lanes(-1)
    plain = [o for o in outs if not o[0]]
    over = [o for o in outs if o[0]]
    for a, b in zip(plain, over):
        assert a[2] == b[2]  # (partial I, partial E, evaluations): bit-identical
        for x, y in zip(a[3], b[3]):
            assert np.array_equal(x, y)


def test_pooled_worker_shell_reused_across_dimensions():
    """Worker shells are pooled across runs; a shell reused for a larger d must
    not keep d-sized scratch (the row staging buffer) from the smaller run."""
    from paper_2511_01573_b200 import _lib
    from paper_2511_01573_b200.regions import partition_arrays
    from paper_2511_01573_b200.worker import DeviceWorker
    _lib.lib().hcub_trim(0)  # empty pool: the d=12 worker below gets the d=2 shell
    for d, rows in ((2, 1100), (12, 1000)):
        dom = hb.HyperRect.unit_cube(d)
        w = DeviceWorker(hb.build_gm_rule(d), hb.make_integrand("f2", d), dom)
        lo, hi = partition_arrays(dom, rows)
        w.append(lo, hi)
        rlo, rhi, _, _, _ = w.read()
        assert np.array_equal(rlo, lo) and np.array_equal(rhi, hi)
        w.close()


def test_overlapped_append_across_row_capacity_keeps_volumes():
    """evaluate_begin -> append -> evaluate_end where the arrivals push the
    store past the per-row scratch capacity (65536 rows on a fresh shell):
    the volumes and split-axis extents K1 wrote for the earlier rows must
    survive the growth, so classify decides exactly as in the
    deliver-then-evaluate order (ensure_rows dropped them)."""
    from paper_2511_01573_b200 import _lib
    from paper_2511_01573_b200.worker import DeviceWorker
    d = 3
    f = hb.make_integrand("f4", d)
    dom = hb.HyperRect.unit_cube(d)
    rng = np.random.default_rng(11)
    n0 = 65536 - 40
    lo = rng.random((n0, d)) * 0.6
    hi = lo + 1e-3 + rng.random((n0, d)) * 0.3
    alo = rng.random((400, d)) * 0.6
    ahi = alo + 1e-3 + rng.random((400, d)) * 0.3
    cfg = hb.DriverConfig(1e-4)
    outs = []
    # one launch shape for both orders (the tail K1 of 400 rows would pick more
    # lanes per region than the full-store K1: same axes, integrals within an ulp)
    hb.set_k1_lanes(0)
    try:
        for overlapped in (False, True):
            _lib.lib().hcub_trim(0)  # fresh shell: rows_cap starts at 65536
            w = DeviceWorker(hb.build_gm_rule(d), f, dom)
            w.append(lo, hi)
            if overlapped:
                w.evaluate_begin()
                w.append(alo, ahi)
                got = w.evaluate_end()
            else:
                w.append(alo, ahi)
                got = w.evaluate()
            oc = w.classify(got[0], cfg)
            outs.append((got, oc, w.read()))
            w.close()
    finally:
        hb.set_k1_lanes(-1)
    (g0, oc0, s0), (g1, oc1, s1) = outs
    assert g0 == g1
    assert oc0 == oc1 and oc0.finalized_count > 0 and oc0.split_count > 0
    for x, y in zip(s0, s1):
        assert np.array_equal(x, y)


def test_capacity_failure_settles_like_reference():
    """A rank whose store cannot hold its split (fixed capacity) ends the run
    with MAX_REGIONS; the settle must count carry + the children's
    provisional halves, as the reference does after its split (ref
    distributed.py:535-537, 406-437) - not carry + the evaluated parents,
    which would count every finalized region twice."""
    from oracle import hcub_oracle as orc
    d = 3
    cap = 1024
    dr = hb.run_distributed(hb.make_integrand("f4", d), hb.HyperRect.unit_cube(d), hb.DriverConfig(1e-6),
                            hb.RedistributionConfig(), workers=1, capacity=cap)
    o = orc.run_distributed(orc.integrand("f4", d), d, 1e-6, 1, max_regions=cap)
    assert dr.result.termination_reason.value == "max_regions" == o.result.termination_reason
    assert dr.result.iterations == o.result.iterations
    assert dr.result.total_f_evals == o.result.total_f_evals
    assert math.isclose(dr.result.integral, o.result.integral, rel_tol=1e-12)
    assert math.isclose(dr.result.error, o.result.error, rel_tol=1e-9)


def test_device_append_rejects_degenerate_rows():
    """On-device appends (the NCCL receive path) validate lo < hi like the
    host path and the reference's append_batch (ref regions.py:204-205)."""
    import torch
    from paper_2511_01573_b200.worker import DeviceWorker
    d = 2
    w = DeviceWorker(hb.build_gm_rule(d), hb.make_integrand("f4", d), hb.HyperRect.unit_cube(d))
    good = torch.tensor([[0.0, 0.0], [0.5, 0.5]], dtype=torch.float64, device="cuda")
    bad = torch.tensor([[0.0, 0.5], [0.5, 0.5]], dtype=torch.float64, device="cuda")  # hi[1] == lo[1]
    w.append_device(good[0:1].data_ptr(), good[1:2].data_ptr(), 1)
    with pytest.raises(ValueError):
        w.append_device(bad[0:1].data_ptr(), bad[1:2].data_ptr(), 1)
    assert len(w) == 1
    w.close()


def test_trace_exception_stops_device_loop():
    """A trace callback that raises stops integrate at that iteration (the
    reference propagates it immediately) instead of after the whole run."""
    calls = []

    def tr(t):
        calls.append(t.iteration)
        if t.iteration == 3:
            raise KeyError("stop")

    with pytest.raises(KeyError):
        hb.integrate(hb.make_integrand("f4", 3), hb.HyperRect.unit_cube(3), hb.DriverConfig(1e-6), trace=tr)
    assert calls == [1, 2, 3]


def test_explicit_split_equals_virtual_children():
    """hcub_worker_classify(split=1) (k3_split materialises the children at
    once - the C-ABI's explicit-split mode) leaves the same store as
    split=2 (virtual children, materialised on read)."""
    import ctypes as C

    from paper_2511_01573_b200 import _lib
    from paper_2511_01573_b200.regions import partition_arrays
    from paper_2511_01573_b200.worker import DeviceWorker
    d = 5
    f = hb.make_integrand("f2", d)
    dom = hb.HyperRect.unit_cube(d)
    cfg = hb.DriverConfig(1e-6)
    stores = []
    for split in (1, 2):
        w = DeviceWorker(hb.build_gm_rule(d), f, dom)
        lo, hi = partition_arrays(dom, 2 * d)
        w.append(lo, hi)
        for it in range(9):
            I, E, _ = w.evaluate()
            out = _lib.hcub_classify_out()
            cd = cfg.descriptor()
            _lib.check(_lib.lib().hcub_worker_classify(w._h, float(I), C.byref(cd), split, C.byref(out)))
            assert out.split_done == 1
        stores.append(w.read()[:2])
        w.close()
    (lo1, hi1), (lo2, hi2) = stores
    assert lo1.shape == lo2.shape and lo1.shape[0] > 1000
    assert np.array_equal(lo1, lo2) and np.array_equal(hi1, hi2)


def test_concurrent_backend_with_degree9_rule():
    """Rank threads building their stores from one shared degree-9 table at the
    same time (descriptor arrays are built once per table) evolve exactly the
    lock-step simulation's run."""
    f = hb.make_product_peak(4, 0.1)[0]
    cfg = hb.DriverConfig(1e-6, rule="gm9")
    dom = hb.HyperRect.unit_cube(4)
    a = hb.run_distributed(f, dom, cfg, workers=4, backend="deterministic_sim", collect_log=True)
    b = hb.run_distributed(f, dom, cfg, workers=4, backend="concurrent", collect_log=True)
    assert a.result.iterations == b.result.iterations and a.result.total_f_evals == b.result.total_f_evals
    assert a.result.integral == b.result.integral and a.result.error == b.result.error
    assert [e["counts"] for e in a.iteration_log] == [e["counts"] for e in b.iteration_log]
    assert a.messages_total == b.messages_total and a.messages_total > 0
