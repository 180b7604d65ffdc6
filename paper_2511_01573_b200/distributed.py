"""Multi-worker adaptive integration with cyclic round-robin redistribution
(ref pkg/src/hcub/distributed.py), on device-resident region stores.

Protocol (identical decisions to the reference on identical inputs):
  per iteration: deliver due batches -> evaluate (K1+K2 on each store) ->
  metadata exchange of per-rank records (the one global sync, rank-ordered
  exact sum, ref :325-346) -> stop test -> classify/split against the global
  integral (K3) -> MAX_REGIONS test -> donors extract their top-error
  regions (K4) for the circle-method partner (ref :253-322) -> census check.

Backends (`run_distributed(backend=...)`):
  deterministic_sim  all ranks in this process (one device or spread over the
                     visible ones), lock-step; TimeBreakdown in the
                     reference's virtual units (evaluations + modeled message
                     cost, ref :492-510) - bit-for-bit the reference's columns.
  concurrent         same in-process lock-step execution, wall-clock
                     per-rank phase times; idle = time a rank would wait at
                     the metadata exchange for the slowest rank.
  nccl               one rank per process (torch.distributed, initialised
                     by the caller, e.g. torchrun): records are all-gathered
                     as one float64 tensor, batches move as device tensors
                     with NCCL send/recv (gloo: host tensors), so region rows
                     never touch the host on the NCCL path.
"""

from __future__ import annotations

import math
import struct
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from .driver import DriverConfig, IntegrationResult, TerminationReason, check_convergence, GlobalEstimate
from .regions import HyperRect, RegionStore, partition_arrays

__all__ = [
    "ProtocolError", "RedistributionConfig", "MetadataRecord", "TransferBatch", "TimeBreakdown", "WorkerState",
    "DistributedResult", "fair_share", "balance_role", "round_robin_pairs", "plan_transfer", "metadata_reduce",
    "run_distributed", "BACKENDS",
]

BACKENDS = ("deterministic_sim", "concurrent", "nccl")


class ProtocolError(RuntimeError):
    """Iteration misalignment or a stalled message (ref distributed.py:72-73)."""


@dataclass(frozen=True)
class RedistributionConfig:
    """ref distributed.py:76-103."""

    cap: int = 512
    initial_subdomains_per_rank: int = 8
    policy: str = "round_robin"
    delivery_latency: int = 1
    max_unacked_iterations: int = 3
    msg_fixed_cost: float = 64.0
    msg_cost_per_region: float = 2.0

    def __post_init__(self):
        if self.cap < 1:
            raise ValueError("cap must be >= 1")
        if self.initial_subdomains_per_rank < 1:
            raise ValueError("initial_subdomains_per_rank must be >= 1")
        if self.policy != "round_robin":
            raise ValueError(f"unknown redistribution policy {self.policy!r}")
        if self.delivery_latency < 1:
            raise ValueError("delivery_latency must be >= 1")


@dataclass(frozen=True)
class MetadataRecord:
    rank: int
    partial_integral: float
    partial_error: float
    inflight_integral_bound: float
    inflight_error_bound: float
    active_count: int

    def as_row(self) -> list[float]:
        return [float(self.rank), self.partial_integral, self.partial_error, self.inflight_integral_bound,
                self.inflight_error_bound, float(self.active_count)]

    @classmethod
    def from_row(cls, row) -> "MetadataRecord":
        return cls(int(row[0]), float(row[1]), float(row[2]), float(row[3]), float(row[4]), int(row[5]))


@dataclass
class TimeBreakdown:
    rank: int
    iterations: int
    compute_seconds: float
    idle_seconds: float
    messages_out: int
    regions_out: int


_WIRE = struct.Struct("<IIQIH")


@dataclass
class TransferBatch:
    """Region coordinates in transit plus the donor's conservative bounds
    (ref distributed.py:133-192); `encode` is the reference's wire format."""

    from_rank: int
    to_rank: int
    sequence_id: int
    lo: np.ndarray
    hi: np.ndarray
    attached_error_bound: float
    attached_integral_bound: float

    @property
    def count(self) -> int:
        return int(self.lo.shape[0])

    @property
    def rects(self) -> list[HyperRect]:
        return [HyperRect(self.lo[i].copy(), self.hi[i].copy()) for i in range(self.count)]

    def encode(self) -> bytes:
        m, d = self.lo.shape
        rows = np.empty((m, 2 * d))
        rows[:, 0::2] = self.lo
        rows[:, 1::2] = self.hi
        return (_WIRE.pack(self.from_rank, self.to_rank, self.sequence_id, m, d) + rows.astype("<f8").tobytes()
                + struct.pack("<dd", self.attached_error_bound, self.attached_integral_bound))

    @classmethod
    def decode(cls, buf: bytes) -> "TransferBatch":
        if len(buf) < _WIRE.size + 16:
            raise ProtocolError("transfer frame truncated")
        frm, to, seq, m, d = _WIRE.unpack_from(buf, 0)
        want = _WIRE.size + 16 * m * d + 16
        if len(buf) != want:
            raise ProtocolError(f"transfer frame has {len(buf)} bytes, expected {want}")
        rows = np.frombuffer(buf, dtype="<f8", count=2 * m * d, offset=_WIRE.size).reshape(m, 2 * d)
        eb, ib = struct.unpack_from("<dd", buf, _WIRE.size + 16 * m * d)
        return cls(frm, to, seq, np.ascontiguousarray(rows[:, 0::2], dtype=np.float64),
                   np.ascontiguousarray(rows[:, 1::2], dtype=np.float64), eb, ib)


# ---------------------------------------------------------------------------
# protocol operations (host decisions, replicated on every rank)


def fair_share(counts: Sequence[int]) -> float:
    counts = list(counts)
    if not counts:
        raise ValueError("need at least one worker")
    return sum(counts) / len(counts)


def balance_role(count: int, share: float) -> str:
    """donor above ceil(share), receiver below floor(share) (ref :245-250)."""
    if count > math.ceil(share):
        return "donor"
    if count < math.floor(share):
        return "receiver"
    return "neutral"


def round_robin_pairs(workers: int, rnd: int) -> list[tuple[int, int]]:
    """Circle-method pairing of round ``rnd`` (ref :253-278): rank 0 meets
    rnd mod (m) + 1, ranks a+1 and b+1 with a + b = 2 rnd (mod m); odd P adds
    a phantom rank that sits out."""
    if workers < 2:
        return []
    n = workers + (workers & 1)
    m = n - 1
    r = rnd % (workers if workers & 1 else workers - 1)
    pairs = [(0, r % m + 1)]
    for a in range(m):
        b = (2 * r - a) % m
        if a < b:
            pairs.append((a + 1, b + 1))
    return [(a, b) for a, b in pairs if a < workers and b < workers]


def _plan(pair, counts, cap):
    """(donor, receiver, n) or None (ref :300-310)."""
    a, b = pair
    share = fair_share(counts)
    ra, rb = balance_role(counts[a], share), balance_role(counts[b], share)
    if {ra, rb} != {"donor", "receiver"}:
        return None
    donor, receiver = (a, b) if ra == "donor" else (b, a)
    n = min(cap, counts[donor] - math.ceil(share), math.floor(share) - counts[receiver])
    return (donor, receiver, n) if n >= 1 else None


TakeTop = Callable[[int, int], tuple]


def plan_transfer(pair, counts, take_top: TakeTop, cfg: RedistributionConfig, sequence_id: int = 0):
    """ref distributed.py:284-322."""
    p = _plan(pair, counts, cfg.cap)
    if p is None:
        return None
    donor, receiver, n = p
    lo, hi, err, integ = take_top(donor, n)
    if lo.shape[0] == 0:
        return None
    return TransferBatch(donor, receiver, sequence_id, lo, hi, math.fsum(np.asarray(err).tolist()),
                         math.fsum(np.abs(np.asarray(integ)).tolist()))


def metadata_reduce(records: Sequence[MetadataRecord], cfg: DriverConfig) -> tuple[float, float, bool]:
    """Rank-ordered exact sums of partials plus in-flight bounds (ref :325-346)."""
    ranks = sorted(r.rank for r in records)
    if ranks != list(range(len(records))):
        raise ProtocolError(f"metadata records misaligned: got ranks {ranks}")
    ordered = sorted(records, key=lambda r: r.rank)
    integral = math.fsum([r.partial_integral for r in ordered] + [r.inflight_integral_bound for r in ordered])
    error = math.fsum([r.partial_error for r in ordered] + [r.inflight_error_bound for r in ordered])
    return integral, error, error <= max(cfg.abs_floor, abs(integral) * cfg.tau_rel)


@dataclass
class DistributedResult:
    result: IntegrationResult
    timings: list[TimeBreakdown]
    messages_total: int
    regions_transferred_total: int
    final_reduce_integral: float = math.nan
    final_reduce_error: float = math.inf
    iteration_log: list[dict] | None = None
    device_stats: dict | None = None  # B200 extra: summed kernel timings / launch counts over ranks


@dataclass
class WorkerState:
    """Per-rank protocol state around a device store (ref :195-225)."""

    rank: int
    worker: object  # DeviceWorker (or a test double with the same operations)
    finalized_integral: float = 0.0
    finalized_error: float = 0.0
    # sequence_id -> (sent_iteration, error_bound, integral_bound, region_count)
    outgoing_in_flight: dict = field(default_factory=dict)
    compute_time: float = 0.0
    idle_time: float = 0.0
    carry_cost: float = 0.0
    messages_out: int = 0
    regions_out: int = 0
    messages_in: int = 0
    regions_in: int = 0
    width_guard_hits: int = 0
    partial: tuple = (0.0, 0.0)

    def inflight_region_count(self) -> int:
        return sum(v[3] for v in self.outgoing_in_flight.values())

    def record(self) -> MetadataRecord:
        return MetadataRecord(self.rank, self.partial[0], self.partial[1],
                              math.fsum(v[2] for v in self.outgoing_in_flight.values()),
                              math.fsum(v[1] for v in self.outgoing_in_flight.values()),
                              len(self.worker))

    @property
    def store(self) -> RegionStore:
        lo, hi, I, E, ax = self.worker.read()
        s = RegionStore(lo.shape[1] if lo.ndim == 2 and lo.shape[0] else getattr(self.worker, "d", 1))
        if lo.shape[0]:
            s.append_batch(lo, hi, I, E, ax)
        return s


# ---------------------------------------------------------------------------
# transports


class _LocalTransport:
    """All ranks in this process."""

    def __init__(self, workers: int):
        self.world = workers
        self.local_ranks = list(range(workers))

    def allgather_records(self, recs: list[MetadataRecord]) -> list[MetadataRecord]:
        return list(recs)

    overlap = False  # transfers complete inside exchange()

    def complete(self) -> None:
        pass

    def allgather_ints(self, rows: list[list[int]]) -> list[list[int]]:
        return [list(r) for r in rows]

    def exchange(self, sends: list[TransferBatch], recvs: list[tuple[int, int, int, int]], states) -> list:
        """sends: batches from local donors; recvs: (from, to, n, seq) expected
        by local receivers.  Wire round-trip like the reference simulator."""
        got = [TransferBatch.decode(b.encode()) for b in sends]
        if sorted((b.from_rank, b.to_rank, b.count) for b in got) != sorted((f, t, n) for f, t, n, _ in recvs):
            raise ProtocolError("transfer plan and delivered batches disagree")
        return got


class _TorchTransport:
    """One rank per process over torch.distributed (NCCL: device tensors)."""

    def __init__(self, d: int):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.local_ranks = [self.rank]
        self.nccl = dist.get_backend() == "nccl"
        self.dev = torch.device("cuda", torch.cuda.current_device()) if self.nccl else torch.device("cpu")
        self.d = d
        self.wait_s = 0.0
        self.overlap = True  # transfers are left in flight across the next K1 launch
        self._pending = []   # p2p work handles of the last exchange
        self._keep = []      # send buffers that must outlive them

    def _gather(self, row):
        torch = self.torch
        t = torch.tensor(row, dtype=torch.float64).to(self.dev, non_blocking=True)
        out = torch.empty(self.world * len(row), dtype=torch.float64, device=self.dev)
        t0 = time.perf_counter()
        self.dist.all_gather_into_tensor(out, t)
        flat = out.cpu().tolist()  # host sync: the decision is replicated on every rank
        self.wait_s += time.perf_counter() - t0
        k = len(row)
        return [flat[i * k:(i + 1) * k] for i in range(self.world)]

    def allgather_records(self, recs):
        return [MetadataRecord.from_row(r) for r in self._gather(recs[0].as_row())]

    def allgather_ints(self, rows):
        return [[int(v) for v in r] for r in self._gather([float(v) for v in rows[0]])]

    def exchange(self, sends, recvs, states):
        """Point-to-point moves of region rows + bounds.  NCCL: the donor's
        rows are gathered straight into a device tensor by K4 and received
        into a device tensor that K5 appends - no host copy."""
        torch, dist = self.torch, self.dist
        ops = []
        keep = []
        for b in sends:  # payload rows (2, m, d) followed by 2 bounds
            if isinstance(b, _DeviceBatch):
                payload = b.payload
            else:
                payload = torch.from_numpy(np.concatenate([b.lo.ravel(), b.hi.ravel(),
                                                           [b.attached_error_bound, b.attached_integral_bound]]))
                payload = payload.to(self.dev)
            keep.append(payload)
            ops.append(dist.P2POp(dist.isend, payload, b.to_rank))
        bufs = []
        for frm, to, n, seq in recvs:
            buf = torch.empty(2 * n * self.d + 2, dtype=torch.float64, device=self.dev)
            bufs.append((frm, to, n, seq, buf))
            ops.append(dist.P2POp(dist.irecv, buf, frm))
        if ops:
            # left in flight: the next iteration launches K1 on the local store
            # first and completes the transfers while it runs (complete())
            self._pending = list(dist.batch_isend_irecv(ops))
            self._keep = keep
        return [_DeviceBatch.from_buffer(frm, to, seq, n, self.d, buf, self.nccl) for frm, to, n, seq, buf in bufs]

    def complete(self) -> None:
        """Wait for the transfers of the last exchange (before delivering)."""
        if self._pending:
            t0 = time.perf_counter()
            for w in self._pending:
                w.wait()
            if self.nccl:
                self.torch.cuda.current_stream().synchronize()
            self.wait_s += time.perf_counter() - t0
        self._pending, self._keep = [], []


class _DeviceBatch:
    """A batch whose rows live in one flat float64 tensor [lo | hi | err_b, int_b]."""

    def __init__(self, from_rank, to_rank, seq, n, d, payload, on_device):
        self.from_rank, self.to_rank, self.sequence_id = from_rank, to_rank, seq
        self.n, self.d, self.payload, self.on_device = n, d, payload, on_device
        self._bounds = None

    def _tail(self):  # read only after the transfer completed (transport.complete())
        if self._bounds is None:
            self._bounds = self.payload[2 * self.n * self.d:].cpu().tolist()
        return self._bounds

    @property
    def attached_error_bound(self):
        return self._tail()[0]

    @property
    def attached_integral_bound(self):
        return self._tail()[1]

    @classmethod
    def from_buffer(cls, frm, to, seq, n, d, buf, on_device):
        return cls(frm, to, seq, n, d, buf, on_device)

    @property
    def count(self):
        return self.n

    @property
    def lo(self):
        return self.payload[: self.n * self.d].reshape(self.n, self.d).cpu().numpy()

    @property
    def hi(self):
        return self.payload[self.n * self.d: 2 * self.n * self.d].reshape(self.n, self.d).cpu().numpy()


# ---------------------------------------------------------------------------
# engine


def _deliver(st: WorkerState, b) -> int:
    """Append a batch at the receiver's tail (ref :400-403); returns the
    first appended row."""
    start = len(st.worker)
    if isinstance(b, _DeviceBatch) and b.on_device:
        base = b.payload.data_ptr()
        st.worker.append_device(base, base + 8 * b.n * b.d, b.n)
    else:
        st.worker.append(b.lo, b.hi)
    st.messages_in += 1
    st.regions_in += b.count
    return start


def _take_batch(st: WorkerState, receiver: int, n: int, seq: int, d: int, transport) -> object | None:
    """K4 on the donor: remove the top-n rows and package them."""
    if isinstance(transport, _TorchTransport) and transport.nccl and hasattr(st.worker, "take_top_device"):
        import torch
        n = min(n, len(st.worker))
        if n <= 0:
            return None
        payload = torch.empty(2 * n * d + 2, dtype=torch.float64, device=transport.dev)
        err = torch.empty(n, dtype=torch.float64, device=transport.dev)
        integ = torch.empty(n, dtype=torch.float64, device=transport.dev)
        base = payload.data_ptr()
        got = st.worker.take_top_device(n, base, base + 8 * n * d, err.data_ptr(), integ.data_ptr())
        eb = math.fsum(err.cpu().tolist())
        ib = math.fsum(integ.abs().cpu().tolist())
        payload[2 * n * d:] = torch.tensor([eb, ib], dtype=torch.float64, device=transport.dev)
        b = _DeviceBatch(st.rank, receiver, seq, got, d, payload, True)
        return b
    lo, hi, err, integ = st.worker.take_top(n)
    if lo.shape[0] == 0:
        return None
    return TransferBatch(st.rank, receiver, seq, lo, hi, math.fsum(err.tolist()),
                         math.fsum(np.abs(integ).tolist()))


def _run(f, domain: HyperRect, cfg: DriverConfig, rcfg: RedistributionConfig, workers: int, backend: str,
         collect_log: bool, make_worker) -> DistributedResult:
    from .rules import get_rule

    table = get_rule(cfg.rule, domain.dim)
    d = domain.dim
    K = table.node_count
    transport = _TorchTransport(d) if backend == "nccl" else _LocalTransport(workers)
    P = transport.world
    if backend == "nccl" and P != workers:
        raise ValueError(f"workers={workers} but the process group has {P} ranks")
    virtual = backend == "deterministic_sim"

    # initial deal: uniform_partition(P * per_rank) -> parts[rank::P] (ref :371-378)
    lo, hi = partition_arrays(domain, P * rcfg.initial_subdomains_per_rank)
    states: dict[int, WorkerState] = {}
    for r in transport.local_ranks:
        w = make_worker(r)
        if lo[r::P].shape[0]:
            w.append(lo[r::P], hi[r::P])
        states[r] = WorkerState(rank=r, worker=w)
    inbox: dict[int, list] = {r: [] for r in transport.local_ranks}  # (deliver_iteration, batch)
    seq_counter = 0  # global batch numbering, derived identically on every rank
    glob_inflight: list[tuple[int, int]] = []  # (sent_iteration, regions) of every unacknowledged batch
    log: list[dict] = []
    total_evals = 0
    peak = P * rcfg.initial_subdomains_per_rank
    expected_census = peak
    virtual_now = 0.0
    iteration = 0
    reason = None
    converged = False
    last = (math.nan, math.inf)

    try:
        while True:
            iteration += 1
            it = iteration - 1
            # liveness guard, acknowledgments due this round (ref :475-489)
            for st in states.values():
                for seq, (sent_it, _, _, _) in st.outgoing_in_flight.items():
                    if it - sent_it > rcfg.max_unacked_iterations:
                        raise ProtocolError(f"batch {seq} from rank {st.rank} unacknowledged for "
                                            f"{it - sent_it} iterations")
                done = [s for s, v in st.outgoing_in_flight.items() if v[0] + rcfg.delivery_latency <= it]
                for s in done:
                    st.outgoing_in_flight.pop(s)
            # evaluation (K1 + exact sums per rank).  Over a process group the
            # last exchange is still in flight: K1 starts on the local store,
            # the transfers complete meanwhile, the arrivals are appended at
            # the tail (ref :482-489 order) and evaluated by a second K1 into
            # the same exact accumulators - identical rows, estimates and sums
            # to delivering first (transfers overlap evaluation).
            overlap = transport.overlap and all(hasattr(st.worker, "evaluate_begin") for st in states.values())
            t_begin = {}
            if overlap:
                for r, st in states.items():
                    t_begin[r] = time.perf_counter()
                    st.worker.evaluate_begin()
            transport.complete()
            for r, box in inbox.items():
                due = sorted((e for e in box if e[0] <= it), key=lambda e: (e[1].from_rank, e[1].sequence_id))
                inbox[r] = [e for e in box if e[0] > it]
                for _, b in due:
                    _deliver(states[r], b)

            work = {}
            for r, st in states.items():
                t0 = t_begin.get(r, time.perf_counter())
                pi, pe, ev = st.worker.evaluate_end() if overlap else st.worker.evaluate()
                st.partial = (pi, pe)
                total_evals += ev
                dt = time.perf_counter() - t0
                work[r] = (ev + st.carry_cost) if virtual else dt
                st.carry_cost = 0.0

            # the one global synchronization point
            mine = [states[r].record() for r in transport.local_ranks]
            records = transport.allgather_records(mine)
            gI, gE, converged = metadata_reduce(records, cfg)
            last = (gI, gE)
            counts = [rec.active_count for rec in records]
            peak = max(peak, sum(counts))
            if isinstance(transport, _LocalTransport):
                # virtual (sim) or modeled-concurrent arrival at the exchange
                arrive = {r: virtual_now + work[r] for r in states}
                now = max(arrive.values())
                for r, st in states.items():
                    st.compute_time += float(work[r])
                    st.idle_time += float(now - arrive[r])
                virtual_now = now
            else:
                for r, st in states.items():
                    st.compute_time += work[r]
            if converged:
                reason = TerminationReason.TOLERANCE
                break
            if iteration >= cfg.max_iterations:
                reason = TerminationReason.MAX_ITERATIONS
                break

            # classify / finalize / split against the global integral (K3)
            local = []
            for r in transport.local_ranks:
                st = states[r]
                t0 = time.perf_counter()
                oc = st.worker.classify(gI, cfg)
                st.finalized_integral, st.finalized_error = oc.finalized_integral, oc.finalized_error
                st.width_guard_hits += oc.width_guard_hits
                st.compute_time += 0.0 if virtual else time.perf_counter() - t0
                local.append([2 * oc.split_count if oc.split_done else -1, oc.finalized_count, oc.split_count])
            allc = transport.allgather_ints(local)
            post_split = [row[0] for row in allc]
            fin_total = sum(row[1] for row in allc)
            split_total = sum(row[2] for row in allc)
            if any(c < 0 or c > cfg.max_regions for c in post_split):
                reason = TerminationReason.MAX_REGIONS
                break

            # redistribution (ref :539-560): plans from the pre-split counts,
            # batches taken from the post-split stores; every rank derives the
            # same schedule, sizes and sequence ids
            sends, recvs, transfers = [], [], []
            for pair in round_robin_pairs(P, it):
                p = _plan(pair, counts, rcfg.cap)
                if p is None:
                    continue
                donor, receiver, n = p
                n = min(n, post_split[donor])
                if n < 1:
                    continue
                seq = seq_counter
                seq_counter += 1
                transfers.append([donor, receiver, n])
                if donor in states:
                    sends.append(_take_batch(states[donor], receiver, n, seq, d, transport))
                if receiver in states:
                    recvs.append((donor, receiver, n, seq))
            arrived = transport.exchange(sends, recvs, states)
            for b in sends:
                st = states[b.from_rank]
                st.outgoing_in_flight[b.sequence_id] = (it, b.attached_error_bound, b.attached_integral_bound,
                                                        b.count)
                st.carry_cost += rcfg.msg_fixed_cost + rcfg.msg_cost_per_region * b.count
                st.messages_out += 1
                st.regions_out += b.count
            for b in arrived:
                inbox[b.to_rank].append((it + rcfg.delivery_latency, b))

            # integer census: nothing lost or duplicated (ref :562-572).  Every
            # rank holds the same global view (post-split counts, transfers,
            # in-flight ledger sizes are replicated), so no extra exchange:
            expected_census = expected_census - fin_total + split_total
            sent = [0] * P
            for donor, receiver, n in transfers:
                sent[donor] += n
            glob_inflight.extend((it, n) for _, _, n in transfers)
            glob_inflight[:] = [(s_it, n) for s_it, n in glob_inflight if s_it + rcfg.delivery_latency > it]
            post_transfer = [post_split[r] - sent[r] for r in range(P)]
            inflight_regions = sum(n for _, n in glob_inflight)
            census = sum(post_transfer) + inflight_regions
            local_ok = all(len(states[r].worker) == post_transfer[r] for r in transport.local_ranks)
            if census != expected_census or not local_ok:
                raise ProtocolError(f"region census broken at iteration {iteration}: {census} present vs "
                                    f"{expected_census} expected")
            if collect_log:
                log.append({
                    "iteration": iteration, "counts": counts, "post_split_counts": post_transfer,
                    "inflight_regions": inflight_regions, "inflight_batches": len(glob_inflight),
                    "transfers": transfers, "global_integral": gI, "global_error": gE, "census": census,
                })
            if census == 0:
                reason = TerminationReason.WIDTH_GUARD_EXHAUSTED
                break

        # settle: deliver and evaluate whatever is still in flight, then one
        # exact sum over every rank's carry and store (ref :406-437)
        extra = 0
        transport.complete()
        for r, box in inbox.items():
            for _, b in sorted(box, key=lambda e: (e[1].from_rank, e[1].sequence_id)):
                start = _deliver(states[r], b)
                extra += states[r].worker.evaluate_tail(start)
        total_evals = sum(row[0] for row in transport.allgather_ints(
            [[total_evals + extra if i == 0 else 0] for i, _ in enumerate(transport.local_ranks)]))
        parts_i = [states[r].worker.exact_partial(0) for r in transport.local_ranks]
        parts_e = [states[r].worker.exact_partial(1) for r in transport.local_ranks]
        settled_i, settled_e = _exact_allreduce(transport, parts_i, parts_e)
        if reason is TerminationReason.WIDTH_GUARD_EXHAUSTED:
            if check_convergence(GlobalEstimate(settled_i, settled_e, settled_i, settled_e, 0), cfg):
                reason, converged = TerminationReason.TOLERANCE, True
        if isinstance(transport, _TorchTransport):
            for st in states.values():
                st.idle_time = transport.wait_s
        timings_local = [[r, states[r].compute_time, states[r].idle_time, states[r].messages_out,
                          states[r].regions_out] for r in transport.local_ranks]
        if isinstance(transport, _TorchTransport):
            rows = transport._gather([float(v) for v in timings_local[0]])
        else:
            rows = timings_local
        timings = [TimeBreakdown(int(row[0]), iteration, float(row[1]), float(row[2]), int(row[3]), int(row[4]))
                   for row in rows]
        res = IntegrationResult(settled_i, settled_e, converged, iteration, total_evals, peak, reason)
        stats = None
        if all(hasattr(states[r].worker, "timings") for r in transport.local_ranks):
            loc = [0.0] * 5
            for r in transport.local_ranks:
                t = states[r].worker.timings()
                loc = [a + b for a, b in zip(loc, [t["k1_ms"], t["k2_ms"], t["k3_ms"], t["k1_launches"],
                                                   t["launches"]])]
            if isinstance(transport, _TorchTransport):
                rows_s = transport._gather(loc)
                loc = [sum(row[i] for row in rows_s) for i in range(5)]
            stats = dict(k1_ms=loc[0], k2_ms=loc[1], k3_ms=loc[2], k1_launches=int(loc[3]), launches=int(loc[4]))
        return DistributedResult(res, timings, sum(t.messages_out for t in timings),
                                 sum(t.regions_out for t in timings), last[0], last[1],
                                 log if collect_log else None, stats)
    finally:
        for st in states.values():
            close = getattr(st.worker, "close", None)
            if close:
                close()


def _exact_allreduce(transport, parts_i, parts_e) -> tuple[float, float]:
    """Exactly rounded sum over all ranks of every carry and store value
    (one rounding, like the reference's single math.fsum)."""
    from .worker import ExactPartial

    tot_i = ExactPartial(0)
    tot_e = ExactPartial(0)
    for p in parts_i:
        tot_i = tot_i + p
    for p in parts_e:
        tot_e = tot_e + p
    if isinstance(transport, _TorchTransport):
        import pickle
        blobs = [None] * transport.world
        transport.dist.all_gather_object(blobs, pickle.dumps((tot_i, tot_e)))
        tot_i = ExactPartial(0)
        tot_e = ExactPartial(0)
        for b in blobs:
            a, e = pickle.loads(b)
            tot_i = tot_i + a
            tot_e = tot_e + e
    return tot_i.rounded(), tot_e.rounded()


def run_distributed(f, domain: HyperRect, cfg: DriverConfig, rcfg: RedistributionConfig | None = None,
                    workers: int = 1, backend: str = "deterministic_sim", collect_log: bool = False, *,
                    make_worker=None, capacity: int = 0) -> DistributedResult:
    """Integrate with ``workers`` cooperating ranks (ref distributed.py:854-877).

    ``backend="nccl"`` needs an initialised torch.distributed process group
    of ``workers`` ranks; each rank's store lives on its current CUDA device.
    ``make_worker(rank)`` overrides the store factory (tests)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    rcfg = rcfg or RedistributionConfig()
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")
    if make_worker is None:
        from . import _lib
        from .rules import get_rule
        from .worker import DeviceWorker

        table = get_rule(cfg.rule, domain.dim)
        if backend == "nccl":
            dev = _lib.current_device()
            make_worker = lambda r: DeviceWorker(table, f, domain, device=dev, capacity=capacity)  # noqa: E731
        else:
            ndev = max(1, _lib.device_count())
            base = _lib.current_device()
            make_worker = lambda r: DeviceWorker(table, f, domain, device=(base + r) % ndev,  # noqa: E731
                                                 capacity=capacity)
    return _run(f, domain, cfg, rcfg, workers, backend, collect_log, make_worker)
