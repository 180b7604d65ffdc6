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
  concurrent         one thread per rank in this process (ref :659-848), rank
                     r on visible device (current + r) mod count; the same
                     protocol code as `nccl` over an in-process collective
                     layer (`_ThreadDist`): records all-gathered, batches moved
                     as device tensors with event-ordered device copies.
                     Wall-clock TimeBreakdown (compute = own phases, idle =
                     waits in the exchange), like the reference's threads.
  nccl               one rank per process (torch.distributed, initialised
                     by the caller, e.g. torchrun): records are all-gathered
                     as one float64 tensor, batches move as device tensors
                     with NCCL send/recv (gloo: host tensors), so region rows
                     never touch the host on the NCCL path.

One collective per iteration: the post-split counts the reference reads
right after classify ride on the next iteration's records (see `_run`).
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
#
# Message format of one scheduled transfer (every transport): the plan fixes
# the size n (rows) on both ends before the donor's split is known, the donor
# fills up to n rows (fewer only if its post-split store is smaller) and a
# 3-word trailer [rows, error bound, integral bound]:
#     [lo (n*d) | hi (n*d) | rows, err_b, int_b]      float64
# so a receiver can post its receive without knowing the donor's post-split
# count - no collective is needed between classify and the transfers.


class _LocalTransport:
    """All ranks in this process, lock-step (deterministic_sim)."""

    overlap = False  # transfers complete inside exchange()
    device_batches = False

    def __init__(self, workers: int):
        self.world = workers
        self.local_ranks = list(range(workers))
        self.wait_s = 0.0

    def allgather_rows(self, rows: list[list[float]]) -> list[list[float]]:
        return [list(r) for r in rows]

    def allgather_ints(self, rows: list[list[int]]) -> list[list[int]]:
        return [[int(v) for v in r] for r in rows]

    def complete(self) -> None:
        pass

    def exchange(self, sends: list, recvs: list[tuple[int, int, int, int]]) -> list:
        """sends: (batch, planned rows) from local donors; recvs: (from, to,
        planned rows, seq) expected by local receivers.  Wire round-trip
        through the reference's frame like its simulator (ref :547-549)."""
        want = {(f, t, q): n for f, t, n, q in recvs}
        got = []
        for b, n in sends:
            if want.pop((b.from_rank, b.to_rank, b.sequence_id), -1) != n or b.count > n:
                raise ProtocolError("transfer plan and delivered batches disagree")
            got.append(TransferBatch.decode(b.encode()))
        if want:
            raise ProtocolError("transfer plan and delivered batches disagree")
        return got


# native NCCL communicators of this process: (group id, rank, world, device) -> handle
_NATIVE_COMMS: dict = {}
# gather staging tensors of this process (_TorchTransport._staging); dropped
# at exit while torch's allocators are still alive (tensors freed during
# interpreter teardown crash in the CUDA host allocator)
_STAGING: dict = {}


def _drop_staging() -> None:
    _STAGING.clear()


import atexit  # noqa: E402

atexit.register(_drop_staging)


def _destroy_native_comms() -> None:
    """Release the cached communicators (callers that tear down their process
    group and keep running may call this; at interpreter exit they are left to
    the driver: destroying them after torch's own NCCL shutdown crashed)."""
    from . import _lib
    for _, h in _NATIVE_COMMS.values():
        _lib.lib().hcub_comm_destroy(h)
    _NATIVE_COMMS.clear()


class _TorchTransport:
    """One rank per process over torch.distributed - NCCL (device tensors) or
    gloo (host tensors) - or one rank per thread over `_ThreadDist` (the
    in-process `concurrent` backend), which has the same interface.

    Per iteration it costs one collective (the metadata records plus the
    previous iteration's split/transfer counts, `_run`) and the point-to-point
    transfers, which stay in flight across the next K1 launch."""

    overlap = True  # transfers are completed after the next K1 launch (complete())

    def __init__(self, d: int, dist=None):
        import torch

        if dist is None:
            import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.local_ranks = [self.rank]
        self.nccl = dist.get_backend() == "nccl"
        self.device_batches = self.nccl
        self.dev = torch.device("cuda", torch.cuda.current_device()) if self.nccl else torch.device("cpu")
        self.d = d
        self.wait_s = 0.0
        self._pending = []   # p2p work handles of the last exchange
        self._keep = []      # send buffers that must outlive them
        self._streams = {}   # worker stream pointer -> torch ExternalStream
        self._own_staging = {}
        # one-sync record exchange (gather_device): device tensors only; over a
        # real process group through this rank's native NCCL communicator
        self.device_records = self.nccl
        self.native = self.nccl and hasattr(dist, "broadcast_object_list")
        self._comm = None

    def _staging(self, dtype, k, pin=None):
        """(host row, device row, device rows, host rows) staging tensors of a
        width-k gather: pinned host memory for device transports.  Over a real
        process group they are kept per process (pinned allocations cost ~1
        ms), so repeated runs reuse them; the in-process thread transport
        keeps its own (its copies run on worker streams that end with the run,
        and it stages through pageable memory: the pinned-memory allocator
        tracks the streams its blocks were used on)."""
        pin = self.nccl if pin is None else pin
        shared = isinstance(self.dist, _ThreadDist) is False
        key = (self.nccl, pin, str(self.dev), dtype, k, self.world, self.rank)
        cache = _STAGING if shared else self._own_staging
        bufs = cache.get(key)
        if bufs is None:
            torch = self.torch
            hs = torch.empty(k, dtype=dtype, pin_memory=pin)
            ho = torch.empty(self.world * k, dtype=dtype, pin_memory=pin)
            if self.nccl:
                ds = torch.empty(k, dtype=dtype, device=self.dev)
                do = torch.empty(self.world * k, dtype=dtype, device=self.dev)
            else:
                ds, do = hs, ho
            bufs = cache[key] = (hs, ds, do, ho)
        return bufs

    def _gather(self, row, dtype=None):
        """all-gather one row per rank -> world rows (host lists).  Staging
        buffers are allocated once per shape: pinned host row -> device ->
        all_gather_into_tensor -> pinned host result, one stream sync."""
        torch = self.torch
        dtype = dtype or torch.float64
        k = len(row)
        hs, ds, do, ho = self._staging(dtype, k)
        hs.numpy()[:] = row
        t0 = time.perf_counter()
        if self.nccl:
            ds.copy_(hs, non_blocking=True)
            self.dist.all_gather_into_tensor(do, ds)
            ho.copy_(do, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:
            self.dist.all_gather_into_tensor(do, ds)
        flat = ho.tolist()
        self.wait_s += time.perf_counter() - t0
        return [flat[i * k:(i + 1) * k] for i in range(self.world)]

    def allgather_rows(self, rows):
        return self._gather(rows[0])

    def _native(self):
        """This rank's native NCCL communicator (hcub_comm_init): created once
        per process group and device (NCCL communicator setup costs ~0.1-1 s)
        and kept for later runs; rank 0's unique id travels over the group."""
        if self._comm is None:
            import ctypes as C

            from . import _lib
            pg = self.dist.distributed_c10d._get_default_group()
            key = (id(pg), self.rank, self.world, self.dev.index)
            entry = _NATIVE_COMMS.get(key)
            # the entry holds the group object itself, so its id cannot be reused by a
            # later group while the communicator is cached
            h = entry[1] if entry is not None and entry[0] is pg else None
            if h is None:
                L = _lib.lib()
                uid = (C.c_ubyte * 128)()
                if self.rank == 0:
                    _lib.check(L.hcub_nccl_unique_id(uid))
                box = [bytes(uid)]
                self.dist.broadcast_object_list(box, src=0)
                uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
                h = C.c_void_p()
                _lib.check(L.hcub_comm_init(self.dev.index, self.rank, self.world, uid, C.byref(h)))
                _NATIVE_COMMS[key] = (pg, h)  # lives until the process exits (see _destroy_native_comms)
            self._comm = h
        return self._comm

    def close(self) -> None:
        self._comm = None  # cached in _NATIVE_COMMS for the next run

    def gather_device(self, worker, row, cfg=None):
        """The one-sync record exchange (device workers, NCCL): the host words
        of `row` go up, the worker copies its partials (columns 1-2) into the
        device row, the rows are all-gathered and, with `cfg`, the global
        integral reduced and classify launched speculatively - all on the
        worker's stream - then the gathered rows come down with one
        synchronisation.  Over a real process group this is one native call
        (hcub_worker_exchange_records on this rank's own NCCL communicator)."""
        if self.native:
            flat = worker.exchange_records(self._native(), self.world, row, _COL_PARTIAL_I, _COL_INFLIGHT_I, cfg)
            k = len(row)
            return [flat[i * k:(i + 1) * k] for i in range(self.world)]
        torch = self.torch
        k = len(row)
        hs, ds, do, ho = self._staging(torch.float64, k, pin=False)
        sp = worker.stream_ptr
        st = self._streams.get(sp)
        if st is None:
            st = self._streams[sp] = torch.cuda.ExternalStream(sp, device=self.dev)
        hs.numpy()[:] = row
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            ds.copy_(hs, non_blocking=True)
            worker.record_partials(ds.data_ptr() + 8 * _COL_PARTIAL_I)
            self.dist.all_gather_into_tensor(do, ds)
            if cfg is not None:
                worker.classify_launch(do.data_ptr(), self.world, k, _COL_PARTIAL_I, _COL_INFLIGHT_I, cfg)
            ho.copy_(do, non_blocking=True)
        st.synchronize()
        flat = ho.tolist()
        self.wait_s += time.perf_counter() - t0
        return [flat[i * k:(i + 1) * k] for i in range(self.world)]

    def allgather_ints(self, rows):
        return [[int(v) for v in r] for r in self._gather([int(v) for v in rows[0]], self.torch.int64)]

    def exchange(self, sends, recvs):
        """Point-to-point moves of region rows + trailer.  NCCL: the donor's
        rows were gathered straight into a device tensor by K4 and are
        received into a device tensor that K5 appends - no host copy."""
        torch, dist = self.torch, self.dist
        ops, keep = [], []
        d = self.d
        for b, n in sends:
            if isinstance(b, _DeviceBatch):
                payload = b.payload
            else:
                buf = np.zeros(2 * n * d + 3)
                m = b.count
                buf[:m * d] = b.lo.ravel()
                buf[n * d:n * d + m * d] = b.hi.ravel()
                buf[2 * n * d:] = (m, b.attached_error_bound, b.attached_integral_bound)
                payload = torch.from_numpy(buf).to(self.dev)
            keep.append(payload)
            ops.append(dist.P2POp(dist.isend, payload, b.to_rank))
        bufs = []
        for frm, to, n, seq in recvs:
            buf = torch.empty(2 * n * d + 3, dtype=torch.float64, device=self.dev)
            bufs.append((frm, to, n, seq, buf))
            ops.append(dist.P2POp(dist.irecv, buf, frm))
        if ops:
            # left in flight: the next iteration launches K1 on the local store
            # first and completes the transfers while it runs (complete())
            self._pending = list(dist.batch_isend_irecv(ops))
            self._keep = keep
        return [_DeviceBatch(frm, to, seq, n, d, buf, self.nccl) for frm, to, n, seq, buf in bufs]

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
    """One transfer message in a flat float64 tensor (format above): n
    planned rows, the trailer says how many are real."""

    def __init__(self, from_rank, to_rank, seq, n, d, payload, on_device, trailer=None):
        self.from_rank, self.to_rank, self.sequence_id = from_rank, to_rank, seq
        self.n, self.d, self.payload, self.on_device = n, d, payload, on_device
        self._trailer = trailer  # known at once on the sending side

    def _tail(self):  # receiving side: read only after the transfer completed (complete())
        if self._trailer is None:
            self._trailer = self.payload[2 * self.n * self.d:].cpu().tolist()
        return self._trailer

    @property
    def count(self) -> int:
        return int(self._tail()[0])

    @property
    def attached_error_bound(self):
        return self._tail()[1]

    @property
    def attached_integral_bound(self):
        return self._tail()[2]

    def row_ptrs(self):
        base = self.payload.data_ptr()
        return base, base + 8 * self.n * self.d

    @property
    def lo(self):
        m = self.count
        return self.payload[: m * self.d].reshape(m, self.d).cpu().numpy()

    @property
    def hi(self):
        m, o = self.count, self.n * self.d
        return self.payload[o: o + m * self.d].reshape(m, self.d).cpu().numpy()


class _Work:
    def __init__(self, fn=None):
        self._fn = fn

    def wait(self):
        if self._fn is not None:
            self._fn()
            self._fn = None
        return True


class _P2POp:
    def __init__(self, op, tensor, peer):
        self.op, self.tensor, self.peer = op, tensor, peer


class _ThreadHub:
    """Rendezvous state shared by the rank threads of one in-process run."""

    def __init__(self, world: int):
        import queue
        import threading

        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self._queue = queue
        self._lock = threading.Lock()
        self._mail = {}
        self.failed = False

    def mailbox(self, src: int, dst: int):
        with self._lock:
            if (src, dst) not in self._mail:
                self._mail[(src, dst)] = self._queue.SimpleQueue()
            return self._mail[(src, dst)]

    def abort(self):
        self.failed = True
        self.barrier.abort()


class _ThreadDist:
    """The subset of torch.distributed `_TorchTransport` uses, for P rank
    threads of one process (backend "concurrent", the reference's threaded
    backend, ref distributed.py:659-848).  backend "nccl": payloads are CUDA
    tensors on each rank's own device, moved with device copies ordered by
    CUDA events (NVLink peer copies between GPUs); "gloo": host tensors.
    Point-to-point messages between a pair are matched in posting order, as
    NCCL's are."""

    def __init__(self, hub: _ThreadHub, rank: int, backend: str):
        self.hub, self.rank, self.backend = hub, rank, backend
        self.P2POp = _P2POp

    def get_world_size(self):
        return self.hub.world

    def get_rank(self):
        return self.rank

    def get_backend(self):
        return self.backend

    @staticmethod
    def isend():  # op markers
        raise NotImplementedError

    @staticmethod
    def irecv():
        raise NotImplementedError

    def barrier(self):
        self.hub.barrier.wait()

    def _rendezvous(self, obj, consume):
        hub = self.hub
        hub.slots[self.rank] = obj
        hub.barrier.wait()
        try:
            consume(list(hub.slots))
        finally:
            hub.barrier.wait()  # nobody re-fills a slot before every rank has read it

    def all_gather_into_tensor(self, out, t):
        import torch

        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

        def consume(parts):
            k = t.numel()
            for i, p in enumerate(parts):
                out[i * k:(i + 1) * k].copy_(p)
            if t.is_cuda:  # the peers' rows are reused once everybody left the rendezvous
                torch.cuda.current_stream(t.device).synchronize()
        self._rendezvous(t, consume)

    def batch_isend_irecv(self, ops):
        import torch

        works = []
        for op in ops:
            if op.op is self.isend:
                payload = op.tensor.clone()  # the receiver owns its copy (sender buffers are reused)
                ev = None
                if payload.is_cuda:
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream(payload.device))
                self.hub.mailbox(self.rank, op.peer).put((payload, ev))
                works.append(_Work())
            else:
                box = self.hub.mailbox(op.peer, self.rank)

                def recv(buf=op.tensor, box=box):
                    while True:
                        try:
                            payload, ev = box.get(timeout=1.0)
                            break
                        except Exception:
                            if self.hub.failed:
                                raise ProtocolError("a peer rank failed") from None
                    if payload.numel() != buf.numel():
                        raise ProtocolError(f"transfer of {payload.numel()} words into a {buf.numel()}-word receive")
                    if ev is not None:
                        torch.cuda.current_stream(buf.device).wait_event(ev)
                    buf.copy_(payload, non_blocking=True)
                works.append(_Work(recv))
        return works


# ---------------------------------------------------------------------------
# engine


def _deliver(st: WorkerState, b) -> int:
    """Append a batch at the receiver's tail (ref :400-403); returns the
    first appended row.  An empty message (the donor's post-split store was
    empty) delivers nothing - the reference sends none (ref :306-307)."""
    start = len(st.worker)
    m = b.count
    if m == 0:
        return start
    if isinstance(b, _DeviceBatch) and b.on_device:
        lo_ptr, hi_ptr = b.row_ptrs()
        st.worker.append_device(lo_ptr, hi_ptr, m)
    else:
        st.worker.append(b.lo, b.hi)
    st.messages_in += 1
    st.regions_in += m
    return start


def _take_batch(st: WorkerState, receiver: int, n: int, seq: int, d: int, transport):
    """K4 on the donor: remove its top-n rows (fewer if the store is smaller)
    and package them as an n-row message."""
    if getattr(transport, "device_batches", False) and hasattr(st.worker, "take_top_device"):
        import torch
        payload = torch.empty(2 * n * d + 3, dtype=torch.float64, device=transport.dev)
        vals = torch.empty(2 * n, dtype=torch.float64, device=transport.dev)
        base = payload.data_ptr()
        got = st.worker.take_top_device(n, base, base + 8 * n * d, vals.data_ptr(), vals.data_ptr() + 8 * n)
        v = vals.cpu().numpy()  # one read for both bounds (exact host sums, ref :316-321)
        eb = math.fsum(v[:got].tolist())
        ib = math.fsum(np.abs(v[n:n + got]).tolist())
        payload[2 * n * d:] = torch.tensor([float(got), eb, ib], dtype=torch.float64)
        return _DeviceBatch(st.rank, receiver, seq, n, d, payload, True, trailer=[got, eb, ib])
    lo, hi, err, integ = st.worker.take_top(n)
    return TransferBatch(st.rank, receiver, seq, lo, hi, math.fsum(np.asarray(err).tolist()),
                         math.fsum(np.abs(np.asarray(integ)).tolist()))


# columns of a gathered record row (MetadataRecord.as_row)
_COL_PARTIAL_I, _COL_INFLIGHT_I = 1, 3

# per-rank words appended to each gathered metadata record: the previous
# iteration's post-split count, finalized count, split count and regions
# sent, plus whether the rank holds spare capacity for splitting all of its
# current rows
_AUX_WORDS = 5


def _run(f, domain: HyperRect, cfg: DriverConfig, rcfg: RedistributionConfig, workers: int, transport,
         virtual: bool, collect_log: bool, make_worker) -> DistributedResult:
    """The protocol loop of one process (all ranks of a lock-step simulation,
    or one rank of a process group / thread group).

    One collective per iteration.  The reference learns every rank's
    post-split count right after classify (for MAX_REGIONS, the transfer
    sizes and the census, ref :521-572); here those counts ride on the NEXT
    iteration's metadata records and the iteration's census and log entry
    are completed then, which is exact because:
      * MAX_REGIONS cannot fire when every rank could split all of its rows:
        2 * count <= max_regions for every rank (the counts are in the
        records) and every rank reserved spare capacity for it (a record
        flag).  Otherwise the counts are exchanged at once, as before;
      * transfer sizes are planned from the pre-split counts (ref :540); the
        donor sends at most that many rows and says how many in the message
        trailer, so receivers post fixed-size receives;
      * a zero census (ref :588-590) means every store is empty and nothing
        is in flight, so the next iteration evaluates nothing; it is detected
        from that iteration's records and the iteration is rolled back."""
    d = domain.dim
    P = transport.world
    if P != workers:
        raise ValueError(f"workers={workers} but the process group has {P} ranks")
    latency = rcfg.delivery_latency

    # initial deal: uniform_partition(P * per_rank) -> parts[rank::P] (ref :371-378)
    lo, hi = partition_arrays(domain, P * rcfg.initial_subdomains_per_rank)
    states: dict[int, WorkerState] = {}
    for r in transport.local_ranks:
        w = make_worker(r)
        if lo[r::P].shape[0]:
            w.append(lo[r::P], hi[r::P])
        states[r] = WorkerState(rank=r, worker=w)
    inbox: dict[int, list] = {r: [] for r in transport.local_ranks}  # (deliver_iteration, batch)
    seq_counter = 0  # batch numbering, derived identically on every rank from the plans
    glob_inflight: list[tuple[int, int]] = []  # (sent_iteration, regions) of every unacknowledged batch
    log: list[dict] = []
    total_evals = 0
    peak = P * rcfg.initial_subdomains_per_rank
    census_box = [peak]  # expected census
    virtual_now = 0.0
    iteration = 0
    reason = None
    converged = False
    last = (math.nan, math.inf)
    pend = None  # the previous iteration, completed from this iteration's records
    fast_eval_s: dict[int, float] = {}  # device evaluation time of one-sync iterations (per rank)

    def eval_delta(st) -> float:
        """Device K1 + sums time since the last call (one-sync iterations)."""
        t = st.worker.timings()
        total = (t["k1_ms"] + t["k2_ms"]) / 1e3
        d = total - fast_eval_s.get(st.rank, 0.0)
        fast_eval_s[st.rank] = total
        return d

    def finish_iteration(pend, aux):
        """Census check and log entry of iteration pend["iteration"] from
        every rank's (post-split, finalized, split, sent) counts."""
        ps = [int(a[0]) for a in aux]
        sent = [int(a[3]) for a in aux]
        census_box[0] = census_box[0] - sum(int(a[1]) for a in aux) + sum(int(a[2]) for a in aux)
        transfers = [[dn, rc, sent[dn]] for dn, rc, _ in pend["planned"] if sent[dn] >= 1]
        pit = pend["it"]
        glob_inflight.extend((pit, n) for _, _, n in transfers)
        glob_inflight[:] = [(s_it, n) for s_it, n in glob_inflight if s_it + latency > pit]
        post_transfer = [ps[r] - sent[r] for r in range(P)]
        inflight_regions = sum(n for _, n in glob_inflight)
        census = sum(post_transfer) + inflight_regions
        if census != census_box[0] or not pend["local_ok"]:
            raise ProtocolError(f"region census broken at iteration {pend['iteration']}: {census} present vs "
                                f"{census_box[0]} expected")
        if collect_log:
            log.append({
                "iteration": pend["iteration"], "counts": pend["counts"], "post_split_counts": post_transfer,
                "inflight_regions": inflight_regions, "inflight_batches": len(glob_inflight),
                "transfers": transfers, "global_integral": pend["gI"], "global_error": pend["gE"],
                "census": census,
            })
        return census

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
                done = [s for s, v in st.outgoing_in_flight.items() if v[0] + latency <= it]
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

            # one-sync path (one rank per process over NCCL, device workers):
            # the partials never visit the host before the exchange - the record
            # row is completed on the device, all-gathered on the worker's stream,
            # the global integral reduced there and classify launched against it
            # speculatively; the host waits once for the gathered records
            fast = (overlap and getattr(transport, "device_records", False) and len(states) == 1
                    and all(hasattr(st.worker, "classify_launch") for st in states.values()))
            final_it = iteration >= cfg.max_iterations
            speculative = False
            work = {}
            for r, st in states.items():
                t0 = t_begin.get(r, time.perf_counter())
                if fast:
                    ev = st.worker.evaluate_end_async()
                    st.partial = (0.0, 0.0)  # filled on the device (record_partials)
                else:
                    pi, pe, ev = st.worker.evaluate_end() if overlap else st.worker.evaluate()
                    st.partial = (pi, pe)
                total_evals += ev
                dt = time.perf_counter() - t0
                work[r] = (ev + st.carry_cost) if virtual else dt
                st.carry_cost = 0.0

            # the one global synchronization point: records + the previous
            # iteration's counts + the spare-capacity flag
            rows = []
            for r in transport.local_ranks:
                w = states[r].worker
                reserve = getattr(w, "reserve", None)
                ok = 1 if reserve is None else int(bool(reserve(2 * len(w))))
                aux = pend["aux"][r] if pend is not None else [0, 0, 0, 0]
                rows.append(states[r].record().as_row() + [float(v) for v in aux] + [float(ok)])
            if fast:
                (r, st), = states.items()
                allrows = transport.gather_device(st.worker, rows[0], None if final_it else cfg)
                speculative = not final_it  # (a final iteration never classifies)
                st.partial = (allrows[r][_COL_PARTIAL_I], allrows[r][_COL_PARTIAL_I + 1])
                # compute = the evaluation's device time (K1 + sums); the rest of
                # the synchronised exchange is the rank's idle time
                if not speculative:  # final iteration: settle its timings now
                    st.worker.classify_discard()
                work[r] = 0.0 if speculative else eval_delta(st)  # else: after commit / discard
            else:
                allrows = transport.allgather_rows(rows)
            records = [MetadataRecord.from_row(x[:6]) for x in allrows]
            aux_all = [x[6:6 + _AUX_WORDS] for x in allrows]
            if pend is not None:
                census = finish_iteration(pend, aux_all)
                pend = None
                if census == 0:
                    # the reference stops at the previous iteration (ref :588-590); since
                    # then nothing was evaluated, delivered or sent
                    iteration -= 1
                    reason = TerminationReason.WIDTH_GUARD_EXHAUSTED
                    if speculative:
                        for st in states.values():
                            st.worker.classify_discard()
                            st.compute_time += eval_delta(st)
                    break
            gI, gE, converged = metadata_reduce(records, cfg)
            if speculative and (converged or iteration >= cfg.max_iterations):
                for st in states.values():
                    st.worker.classify_discard()
                    work[st.rank] = eval_delta(st)
            last = (gI, gE)
            counts = [rec.active_count for rec in records]
            peak = max(peak, sum(counts))
            if virtual:
                # virtual arrival at the exchange (ref :506-510)
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
            local = {}
            for r in transport.local_ranks:
                st = states[r]
                t0 = time.perf_counter()
                if speculative:
                    oc = st.worker.classify_commit(gI, cfg)
                    st.compute_time += eval_delta(st)
                else:
                    oc = st.worker.classify(gI, cfg)
                st.finalized_integral, st.finalized_error = oc.finalized_integral, oc.finalized_error
                st.width_guard_hits += oc.width_guard_hits
                st.compute_time += 0.0 if virtual else time.perf_counter() - t0
                local[r] = [2 * oc.split_count if oc.split_done else -1, oc.finalized_count, oc.split_count]
            safe = all(a[4] > 0 for a in aux_all) and 2 * max(counts) <= cfg.max_regions
            allc = None
            if not safe:  # a split may overflow: learn every post-split count now (ref :535-537)
                allc = transport.allgather_ints([local[r] for r in transport.local_ranks])
                if any(row[0] < 0 or row[0] > cfg.max_regions for row in allc):
                    reason = TerminationReason.MAX_REGIONS
                    break

            # redistribution (ref :539-560): plans from the pre-split counts,
            # batches taken from the post-split stores
            sends, recvs, planned = [], [], []
            for pair in round_robin_pairs(P, it):
                p = _plan(pair, counts, rcfg.cap)
                if p is None:
                    continue
                donor, receiver, n = p
                if allc is not None:
                    n = min(n, allc[donor][0])
                    if n < 1:
                        continue
                seq = seq_counter
                seq_counter += 1
                planned.append((donor, receiver, n))
                if donor in states:
                    sends.append((_take_batch(states[donor], receiver, n, seq, d, transport), n))
                if receiver in states:
                    recvs.append((donor, receiver, n, seq))
            arrived = transport.exchange(sends, recvs)
            sent_local = {r: 0 for r in transport.local_ranks}
            for b, _ in sends:
                if b.count == 0:
                    continue  # nothing to send: no message in the reference (ref :306-307)
                st = states[b.from_rank]
                st.outgoing_in_flight[b.sequence_id] = (it, b.attached_error_bound, b.attached_integral_bound,
                                                        b.count)
                st.carry_cost += rcfg.msg_fixed_cost + rcfg.msg_cost_per_region * b.count
                st.messages_out += 1
                st.regions_out += b.count
                sent_local[b.from_rank] = b.count
            for b in arrived:
                inbox[b.to_rank].append((it + latency, b))
            pend = dict(it=it, iteration=iteration, counts=counts, gI=gI, gE=gE, planned=planned,
                        aux={r: local[r] + [sent_local[r]] for r in transport.local_ranks},
                        local_ok=all(len(states[r].worker) == local[r][0] - sent_local[r]
                                     for r in transport.local_ranks))
            if allc is not None:  # every count is known already: finish now (ref :562-590)
                sent_all = [0] * P
                for dn, _, n in planned:  # n <= the donor's post-split count: all of it moves
                    sent_all[dn] = n
                census = finish_iteration(pend, [[allc[r][0], allc[r][1], allc[r][2], sent_all[r]]
                                                 for r in range(P)])
                pend = None
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
        ev_rows = transport.allgather_ints([[total_evals + extra if i == 0 else 0]
                                            for i, _ in enumerate(transport.local_ranks)])
        total_evals = sum(row[0] for row in ev_rows)
        parts_i = [states[r].worker.exact_partial(0) for r in transport.local_ranks]
        parts_e = [states[r].worker.exact_partial(1) for r in transport.local_ranks]
        settled_i, settled_e = _exact_allreduce(transport, parts_i, parts_e)
        if reason is TerminationReason.WIDTH_GUARD_EXHAUSTED:
            if check_convergence(GlobalEstimate(settled_i, settled_e, settled_i, settled_e, 0), cfg):
                reason, converged = TerminationReason.TOLERANCE, True
        if not virtual:
            for st in states.values():
                # (one-sync exchanges also waited for the evaluation itself)
                st.idle_time = max(0.0, transport.wait_s - fast_eval_s.get(st.rank, 0.0))
        rows = transport.allgather_rows([[r, states[r].compute_time, states[r].idle_time, states[r].messages_out,
                                          states[r].regions_out] for r in transport.local_ranks])
        timings = [TimeBreakdown(int(row[0]), iteration, float(row[1]), float(row[2]), int(row[3]), int(row[4]))
                   for row in rows]
        res = IntegrationResult(settled_i, settled_e, converged, iteration, total_evals, peak, reason)
        stats = None
        if all(hasattr(states[r].worker, "timings") for r in transport.local_ranks):
            loc = []
            for r in transport.local_ranks:
                t = states[r].worker.timings()
                loc.append([t["k1_ms"], t["k2_ms"], t["k3_ms"], t["k1_launches"], t["launches"]])
            rows_s = transport.allgather_rows(loc)
            tot = [sum(row[i] for row in rows_s) for i in range(5)]
            stats = dict(k1_ms=tot[0], k2_ms=tot[1], k3_ms=tot[2], k1_launches=int(tot[3]), launches=int(tot[4]))
        return DistributedResult(res, timings, sum(t.messages_out for t in timings),
                                 sum(t.regions_out for t in timings), last[0], last[1],
                                 log if collect_log else None, stats)
    finally:
        for st in states.values():
            close = getattr(st.worker, "close", None)
            if close:
                close()


_PARTIAL_BYTES = 288  # |value| < 2^2176: a sum of < 2^40 finite doubles in units of 2^-1074


def _partial_words(p) -> list[int]:
    words = list(struct.unpack(f"<{_PARTIAL_BYTES // 8}q", p.value.to_bytes(_PARTIAL_BYTES, "little", signed=True)))
    return words + [p.nan, p.pinf, p.ninf]


def _partial_from_words(words):
    from .worker import ExactPartial

    k = _PARTIAL_BYTES // 8
    v = int.from_bytes(struct.pack(f"<{k}q", *[int(x) for x in words[:k]]), "little", signed=True)
    return ExactPartial(v, int(words[k]), int(words[k + 1]), int(words[k + 2]))


def _exact_allreduce(transport, parts_i, parts_e) -> tuple[float, float]:
    """Exactly rounded sum over all ranks of every carry and store value
    (one rounding, like the reference's single math.fsum, ref :430-437).
    The exact per-rank partials travel as fixed-width integer words."""
    from .worker import ExactPartial

    tot_i, tot_e = ExactPartial(0), ExactPartial(0)
    for p in parts_i:
        tot_i = tot_i + p
    for p in parts_e:
        tot_e = tot_e + p
    if not isinstance(transport, _LocalTransport):
        k = len(_partial_words(tot_i))
        rows = transport.allgather_ints([_partial_words(tot_i) + _partial_words(tot_e)])
        tot_i, tot_e = ExactPartial(0), ExactPartial(0)
        for row in rows:
            tot_i = tot_i + _partial_from_words(row[:k])
            tot_e = tot_e + _partial_from_words(row[k:])
    return tot_i.rounded(), tot_e.rounded()


def _run_threads(f, domain, cfg, rcfg, workers, collect_log, make_worker, device_tensors, devices):
    """backend "concurrent": one thread per rank (ref :659-848), each running
    the process-group protocol over `_ThreadDist`.  The C library releases
    the GIL, so the ranks' K1/K3 launches and host waits overlap - across
    GPUs when the ranks sit on different devices."""
    import threading

    hub = _ThreadHub(workers)
    out = [None] * workers
    errors = []

    def body(r):
        try:
            if device_tensors:
                import torch
                torch.cuda.set_device(devices[r])
            tr = _TorchTransport(domain.dim, dist=_ThreadDist(hub, r, "nccl" if device_tensors else "gloo"))
            out[r] = _run(f, domain, cfg, rcfg, workers, tr, False, collect_log, make_worker)
        except BaseException as exc:  # noqa: BLE001 - re-raised on the caller's thread
            errors.append((r, exc))
            hub.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"hcub-rank{r}", daemon=True) for r in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        import threading as _th
        first = [e for _, e in errors if not isinstance(e, _th.BrokenBarrierError)] or [errors[0][1]]
        raise first[0]
    return out[0]


def run_distributed(f, domain: HyperRect, cfg: DriverConfig, rcfg: RedistributionConfig | None = None,
                    workers: int = 1, backend: str = "deterministic_sim", collect_log: bool = False, *,
                    make_worker=None, capacity: int = 0) -> DistributedResult:
    """Integrate with ``workers`` cooperating ranks (ref distributed.py:854-877).

    ``backend="nccl"`` needs an initialised torch.distributed process group
    of ``workers`` ranks; each rank's store lives on its current CUDA device.
    ``backend="concurrent"`` runs one thread per rank in this process, rank r
    on visible device (current + r) mod count.  ``make_worker(rank)``
    overrides the store factory (tests; host-memory transfers then)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    rcfg = rcfg or RedistributionConfig()
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")
    device_tensors = make_worker is None
    devices = None
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
            devices = [(base + r) % ndev for r in range(workers)]
            make_worker = lambda r: DeviceWorker(table, f, domain, device=devices[r],  # noqa: E731
                                                 capacity=capacity)
    if backend == "concurrent":
        return _run_threads(f, domain, cfg, rcfg, workers, collect_log, make_worker, device_tensors, devices)
    transport = _TorchTransport(domain.dim) if backend == "nccl" else _LocalTransport(workers)
    try:
        return _run(f, domain, cfg, rcfg, workers, transport, backend == "deterministic_sim", collect_log, make_worker)
    finally:
        close = getattr(transport, "close", None)
        if close:
            close()
