"""Host protocol of run_distributed (CPU): the engine driven by oracle-backed
workers must reproduce the reference's own deterministic_sim logs exactly -
per-iteration counts, post-split counts, transfers (donor, receiver, size),
census, virtual compute/idle columns and the settled result.  The same
engine over a gloo process group (world size 2, one rank per process) must
produce the in-process result."""
import math
import os
import socket

import numpy as np
import pytest

from conftest import domain_of, golden_names, load_json
from oracle_worker import factory

import paper_2511_01573_b200 as hb
from paper_2511_01573_b200 import distributed as dist_mod

DIST = [n for n in golden_names("dist")]


def spec_inputs(spec):
    d = spec["d"]
    dlo, dhi = domain_of(spec)
    cfg = hb.DriverConfig(spec["tau"])
    rcfg = hb.RedistributionConfig(cap=spec.get("cap", 512), initial_subdomains_per_rank=spec.get("per_rank", 8),
                                   delivery_latency=spec.get("latency", 1))
    return d, dlo, dhi, cfg, rcfg


@pytest.mark.parametrize("name", [n for n in DIST if n.startswith(("f4", "f3", "f6")) or "P3" in n or "cap16" in n
                                  or "lat" in n])
def test_engine_matches_reference_sim_logs(name):
    g = load_json("dist", name)
    spec = g["spec"]
    d, dlo, dhi, cfg, rcfg = spec_inputs(spec)
    dr = hb.run_distributed(None, hb.HyperRect(dlo, dhi), cfg, rcfg, workers=spec["P"], collect_log=True,
                            make_worker=factory(spec, dlo, dhi))
    res = g["result"]
    assert dr.result.termination_reason.value == res["termination_reason"]
    assert dr.result.iterations == res["iterations"]
    assert dr.result.total_f_evals == res["total_f_evals"]
    assert dr.result.peak_regions == res["peak_regions"]
    assert dr.result.integral == res["integral"]  # oracle workers: bit-identical numerics
    assert dr.result.error == res["error"]
    assert dr.messages_total == g["messages_total"]
    assert dr.regions_transferred_total == g["regions_transferred_total"]
    assert dr.final_reduce_integral == g["final_reduce_integral"]
    assert len(dr.iteration_log) == len(g["log"])
    for mine, ref in zip(dr.iteration_log, g["log"]):
        for key in ("counts", "post_split_counts", "inflight_regions", "inflight_batches", "census",
                    "global_integral", "global_error"):
            assert mine[key] == ref[key], (key, mine["iteration"])
        assert [list(t) for t in mine["transfers"]] == [list(t) for t in ref["transfers"]]
    for t, rt in zip(dr.timings, g["timings"]):
        assert (t.rank, t.iterations, t.compute_seconds, t.idle_seconds, t.messages_out, t.regions_out) == \
               (rt["rank"], rt["iterations"], rt["compute"], rt["idle"], rt["messages_out"], rt["regions_out"])


def test_protocol_helpers_match_reference_spec_examples():
    # SPEC.md fair_share / roles / circle schedule
    assert hb.fair_share([10, 2, 6]) == 6.0
    assert dist_mod.balance_role(10, 6.0) == "donor" and dist_mod.balance_role(2, 6.0) == "receiver"
    assert dist_mod.balance_role(6, 6.0) == "neutral"
    assert hb.round_robin_pairs(4, 0) == [(0, 1), (2, 3)]
    assert hb.round_robin_pairs(1, 5) == []
    from oracle import hcub_oracle as orc
    for P in range(2, 11):
        for r in range(12):
            assert hb.round_robin_pairs(P, r) == orc.rr_pairs(P, r)


def test_wire_codec_roundtrip_and_framing():
    b = hb.TransferBatch(1, 2, 7, np.arange(6.0).reshape(3, 2), np.arange(6.0).reshape(3, 2) + 1, 0.5, 1.5)
    w = b.encode()
    assert len(w) == 22 + 3 * 2 * 2 * 8 + 16
    c = hb.TransferBatch.decode(w)
    assert np.array_equal(c.lo, b.lo) and np.array_equal(c.hi, b.hi) and c.sequence_id == 7
    with pytest.raises(hb.ProtocolError):
        hb.TransferBatch.decode(w[:-1])


def test_metadata_reduce_misaligned():
    cfg = hb.DriverConfig(1e-3)
    recs = [hb.MetadataRecord(0, 1.0, 0.1, 0, 0, 3), hb.MetadataRecord(2, 1.0, 0.1, 0, 0, 3)]
    with pytest.raises(hb.ProtocolError):
        hb.metadata_reduce(recs, cfg)
    I, E, conv = hb.metadata_reduce([hb.MetadataRecord(1, 2.0, 1e-9, 0, 0, 1), hb.MetadataRecord(0, 1.0, 1e-9, 0, 0, 1)], cfg)
    assert (I, E, conv) == (3.0, 2e-9, True)


def test_latency_two_and_liveness_guard():
    """delivery_latency > 1 exercises the in-flight bounds; latency beyond
    max_unacked_iterations trips the liveness guard (ref :475-481)."""
    spec = {"f": "pp", "d": 3, "center": 0.1, "tau": 1e-4, "P": 2}
    d, dlo, dhi, cfg, _ = spec_inputs(spec)
    from oracle import hcub_oracle as orc
    dr = hb.run_distributed(None, hb.HyperRect(dlo, dhi), cfg, hb.RedistributionConfig(delivery_latency=2),
                            workers=2, collect_log=True, make_worker=factory(spec, dlo, dhi))
    assert dr.result.termination_reason == hb.TerminationReason.TOLERANCE
    assert any(e["inflight_regions"] > 0 for e in dr.iteration_log) or dr.messages_total == 0
    exact = orc.product_peak(3, 0.1)
    with pytest.raises(hb.ProtocolError):
        hb.run_distributed(None, hb.HyperRect(dlo, dhi), hb.DriverConfig(1e-7),
                           hb.RedistributionConfig(delivery_latency=5, max_unacked_iterations=3, cap=4),
                           workers=2, make_worker=factory(spec, dlo, dhi))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_rank(rank, world, port, name, out, overlap=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_json("dist", name)
        spec = g["spec"]
        d, dlo, dhi, cfg, rcfg = spec_inputs(spec)
        dr = hb.run_distributed(None, hb.HyperRect(dlo, dhi), cfg, rcfg, workers=world, backend="nccl",
                                collect_log=True, make_worker=factory(spec, dlo, dhi, overlap))
        out.put((rank, dr.result.integral, dr.result.error, dr.result.iterations, dr.result.total_f_evals,
                 dr.messages_total, dr.regions_transferred_total,
                 [(e["counts"], e["transfers"], e["census"]) for e in dr.iteration_log]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True], ids=["deliver_first", "overlapped"])
@pytest.mark.parametrize("name", ["pp_d4_c01_P2", "f4_d3_P2"])
def test_gloo_world2_matches_reference(name, overlap):
    """Two ranks over gloo reproduce the reference simulator's log - with the
    transfers completed before evaluation, and left in flight across the next
    evaluation (arrivals appended at the tail and evaluated last)."""
    import multiprocessing as mp
    g = load_json("dist", name)
    if g["spec"]["P"] != 2:
        pytest.skip("world size 2 only")
    if g["wall_s"] if "wall_s" in g else False:
        pass
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, name, q, overlap)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    res = g["result"]
    for o in outs:
        if overlap:  # the oracle's BLAS rounding depends on the batch split (not the device's)
            assert math.isclose(o[1], res["integral"], rel_tol=1e-12)
            assert math.isclose(o[2], res["error"], rel_tol=1e-12)
        else:
            assert o[1] == res["integral"] and o[2] == res["error"]
        assert o[3] == res["iterations"] and o[4] == res["total_f_evals"]
        assert o[5] == g["messages_total"] and o[6] == g["regions_transferred_total"]
        assert [(c, [list(t) for t in tr], ce) for c, tr, ce in o[7]] == \
               [(e["counts"], [list(t) for t in e["transfers"]], e["census"]) for e in g["log"]]


@pytest.mark.parametrize("overlap", [False, True], ids=["deliver_first", "overlapped"])
@pytest.mark.parametrize("name", ["pp_d4_c01_P3", "pp_d4_c01_P4_lat2", "pp_d4_c01_P8_lat2_cap16", "f6_d3_P4_lat2",
                                  "f3_d4_P4"])
def test_concurrent_threads_match_reference(name, overlap):
    """backend="concurrent": one thread per rank, each running the process-group
    protocol (`_TorchTransport` over the in-process `_ThreadDist`, host
    tensors here) - the reference's threaded backend (ref :659-848).  Same
    region flow as the reference's simulator: counts, post-split counts,
    transfers, in-flight ledger, census, settled result."""
    g = load_json("dist", name)
    spec = g["spec"]
    d, dlo, dhi, cfg, rcfg = spec_inputs(spec)
    dr = hb.run_distributed(None, hb.HyperRect(dlo, dhi), cfg, rcfg, workers=spec["P"], backend="concurrent",
                            collect_log=True, make_worker=factory(spec, dlo, dhi, overlap))
    res = g["result"]
    assert dr.result.termination_reason.value == res["termination_reason"]
    assert (dr.result.iterations, dr.result.total_f_evals, dr.result.peak_regions) == \
           (res["iterations"], res["total_f_evals"], res["peak_regions"])
    assert math.isclose(dr.result.integral, res["integral"], rel_tol=1e-12)
    assert math.isclose(dr.result.error, res["error"], rel_tol=1e-12)
    assert (dr.messages_total, dr.regions_transferred_total) == (g["messages_total"], g["regions_transferred_total"])
    assert len(dr.iteration_log) == len(g["log"])
    for mine, ref in zip(dr.iteration_log, g["log"]):
        for key in ("counts", "post_split_counts", "inflight_regions", "inflight_batches", "census"):
            assert mine[key] == ref[key], (key, mine["iteration"])
        assert [list(t) for t in mine["transfers"]] == [list(t) for t in ref["transfers"]]
        assert math.isclose(mine["global_error"], ref["global_error"], rel_tol=1e-12)
    assert [t.rank for t in dr.timings] == list(range(spec["P"]))
    assert all(t.compute_seconds > 0 for t in dr.timings)


def test_concurrent_threads_failure_propagates():
    """An exception on one rank thread ends the run with that exception on
    the caller (the peers' barriers are broken, ref :790-792)."""
    spec = {"f": "pp", "d": 3, "center": 0.1, "tau": 1e-4, "P": 3}
    d, dlo, dhi, cfg, rcfg = spec_inputs(spec)
    make = factory(spec, dlo, dhi)

    class Boom(Exception):
        pass

    def make_worker(r):
        w = make(r)
        if r == 1:
            real = w.classify
            calls = []

            def classify(gI, cfg):
                calls.append(1)
                if len(calls) == 3:
                    raise Boom("rank 1")
                return real(gI, cfg)
            w.classify = classify
        return w

    with pytest.raises(Boom):
        hb.run_distributed(None, hb.HyperRect(dlo, dhi), cfg, rcfg, workers=3, backend="concurrent",
                           make_worker=make_worker)


@pytest.mark.parametrize("P,max_regions", [(2, 300), (3, 150)])
def test_max_regions_immediate_exchange_matches_oracle(P, max_regions):
    """When a split may overflow max_regions the post-split counts are
    exchanged at once (ref :535-537) - the exact fallback of the lazy
    bookkeeping - in the simulator and over the thread transport."""
    from oracle import hcub_oracle as orc
    spec = {"f": "f4", "d": 3, "tau": 1e-7, "P": P}
    d, dlo, dhi, _, rcfg = spec_inputs(spec)
    cfg = hb.DriverConfig(1e-7, max_regions=max_regions)
    o = orc.run_distributed(orc.integrand("f4", 3), 3, 1e-7, P, max_regions=max_regions)
    for backend in ("deterministic_sim", "concurrent"):
        dr = hb.run_distributed(None, hb.HyperRect(dlo, dhi), cfg, rcfg, workers=P, backend=backend,
                                collect_log=True, make_worker=factory(spec, dlo, dhi))
        assert dr.result.termination_reason.value == o.result.termination_reason == "max_regions"
        assert dr.result.iterations == o.result.iterations
        assert dr.result.total_f_evals == o.result.total_f_evals
        assert math.isclose(dr.result.integral, o.result.integral, rel_tol=1e-13)
        assert [e["counts"] for e in dr.iteration_log] == [e["counts"] for e in o.log]
