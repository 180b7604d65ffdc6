"""One region store on one device: the unit a rank of `run_distributed` owns
(ref pkg/src/hcub/distributed.py:195-225 WorkerState.store).

`DeviceWorker` wraps the C-ABI `hcub_worker_*` entry points: the store lives
in HBM (SoA lo/hi/integral/error), evaluation is K1 (+K2), classification and
bisection K3, top-n extraction K4, appends K5.  Rows cross to the host only
for transfers in host-memory transports and for explicit snapshots.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib

SCALE_BITS = 1074  # superaccumulator unit: 2^-1074


@dataclass
class ClassifyResult:
    """ref driver.py:137-144 ClassifyOutcome (store stays on the device)."""

    finalized_integral: float
    finalized_error: float
    width_guard_hits: int
    finalized_count: int
    split_count: int
    children_integral: float
    children_error: float
    split_done: bool


@dataclass
class ExactPartial:
    """carry + sum(column) as an exact integer in units of 2^-1074 plus
    special-value counts (nan, +inf, -inf)."""

    value: int
    nan: int = 0
    pinf: int = 0
    ninf: int = 0

    def __add__(self, other: "ExactPartial") -> "ExactPartial":
        return ExactPartial(self.value + other.value, self.nan + other.nan, self.pinf + other.pinf,
                            self.ninf + other.ninf)

    @staticmethod
    def of(x: float) -> "ExactPartial":
        if x != x:
            return ExactPartial(0, nan=1)
        if x in (float("inf"), float("-inf")):
            return ExactPartial(0, pinf=int(x > 0), ninf=int(x < 0))
        return ExactPartial(int(Fraction(x) * (1 << SCALE_BITS)))

    def rounded(self) -> float:
        """Correctly rounded value, math.fsum semantics for specials."""
        if self.nan or (self.pinf and self.ninf):
            return float("nan")
        if self.pinf:
            return float("inf")
        if self.ninf:
            return float("-inf")
        return float(Fraction(self.value, 1 << SCALE_BITS))


class DeviceWorker:
    """A device-resident region store with the protocol operations."""

    def __init__(self, table, f, domain, device: int | None = None, capacity: int = 0):
        from .integrands import device_descriptor

        self.d = domain.dim
        self.K = table.node_count
        self.device = _lib.current_device() if device is None else int(device)
        self._rd = table.descriptor()
        self._fd = device_descriptor(f, self.d)
        dlo = np.ascontiguousarray(domain.lo, dtype=np.float64)
        dhi = np.ascontiguousarray(domain.hi, dtype=np.float64)
        h = C.c_void_p()
        _lib.check(_lib.lib().hcub_worker_create(self.device, C.byref(self._rd), C.byref(self._fd), _lib.dptr(dlo),
                                                 _lib.dptr(dhi), int(capacity), C.byref(h)))
        self._h = h

    # -- lifecycle -----------------------------------------------------------
    def close(self):
        if self._h:
            _lib.lib().hcub_worker_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- store ---------------------------------------------------------------
    def __len__(self) -> int:
        n = C.c_int64(0)
        _lib.check(_lib.lib().hcub_worker_size(self._h, C.byref(n), None))
        return int(n.value)

    def append(self, lo, hi, integral=None, error=None):
        lo = np.ascontiguousarray(np.atleast_2d(lo), dtype=np.float64)
        hi = np.ascontiguousarray(np.atleast_2d(hi), dtype=np.float64)
        if lo.shape != hi.shape or (lo.size and lo.shape[1] != self.d):
            raise ValueError("bounds shape mismatch")
        iv = None if integral is None else np.ascontiguousarray(integral, dtype=np.float64)
        ev = None if error is None else np.ascontiguousarray(error, dtype=np.float64)
        _lib.check(_lib.lib().hcub_worker_append(self._h, _lib.dptr(lo), _lib.dptr(hi), _lib.dptr(iv), _lib.dptr(ev),
                                                 lo.shape[0] if lo.size else 0, 0))

    def append_device(self, lo_ptr: int, hi_ptr: int, m: int):
        """rows (m, d) already in device memory (e.g. an NCCL receive buffer)."""
        D = _lib._D
        _lib.check(_lib.lib().hcub_worker_append(self._h, C.cast(lo_ptr, D), C.cast(hi_ptr, D), None, None, int(m), 1))

    def read(self):
        n = len(self)
        lo = np.empty((n, self.d))
        hi = np.empty((n, self.d))
        I = np.empty(n)
        E = np.empty(n)
        ax = np.empty(n, dtype=np.int64)
        if n:
            _lib.check(_lib.lib().hcub_worker_read(self._h, _lib.dptr(lo), _lib.dptr(hi), _lib.dptr(I), _lib.dptr(E),
                                                   _lib.iptr(ax)))
        return lo, hi, I, E, ax

    # -- carry ---------------------------------------------------------------
    @property
    def carry(self) -> tuple[float, float]:
        a, b = C.c_double(), C.c_double()
        _lib.check(_lib.lib().hcub_worker_get_carry(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    @carry.setter
    def carry(self, v):
        _lib.check(_lib.lib().hcub_worker_set_carry(self._h, float(v[0]), float(v[1])))

    # -- protocol operations -------------------------------------------------
    def evaluate(self) -> tuple[float, float, int]:
        """K1 over the store; partials = fsum([carry, *column]) (ref
        distributed.py:217-225)."""
        pi, pe, ev = C.c_double(), C.c_double(), C.c_int64()
        _lib.check(_lib.lib().hcub_worker_evaluate(self._h, C.byref(pi), C.byref(pe), C.byref(ev)))
        return pi.value, pe.value, int(ev.value)

    def evaluate_begin(self) -> None:
        """Launch K1 over the store and return at once; rows appended before
        evaluate_end() are evaluated there into the same exact sums."""
        _lib.check(_lib.lib().hcub_worker_evaluate_begin(self._h))

    def evaluate_end(self) -> tuple[float, float, int]:
        pi, pe, ev = C.c_double(), C.c_double(), C.c_int64()
        _lib.check(_lib.lib().hcub_worker_evaluate_end(self._h, C.byref(pi), C.byref(pe), C.byref(ev)))
        return pi.value, pe.value, int(ev.value)

    # -- one-sync protocol (distributed.py over NCCL) ------------------------
    def evaluate_end_async(self) -> int:
        """evaluate_end() without the host read: the partials stay on the
        device (record_partials); returns the evaluation count."""
        ev = C.c_int64()
        _lib.check(_lib.lib().hcub_worker_evaluate_end_async(self._h, C.byref(ev)))
        return int(ev.value)

    @property
    def stream_ptr(self) -> int:
        s = C.c_void_p()
        _lib.check(_lib.lib().hcub_worker_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def record_partials(self, dev_ptr: int) -> None:
        _lib.check(_lib.lib().hcub_worker_record_partials(self._h, C.c_void_p(dev_ptr)))

    def classify_launch(self, rows_ptr: int, ranks: int, width: int, col_integral: int, col_bound: int, cfg) -> None:
        self._cd = cfg.descriptor()
        _lib.check(_lib.lib().hcub_worker_classify_launch(self._h, C.c_void_p(rows_ptr), int(ranks), int(width),
                                                          int(col_integral), int(col_bound), C.byref(self._cd)))

    def exchange_records(self, comm, world: int, row, col_partial: int, col_bound: int, cfg=None) -> list:
        """hcub_worker_exchange_records: all-gather of the record rows over the
        native communicator (+ speculative classify with cfg) -> flat list."""
        r = np.ascontiguousarray(row, dtype=np.float64)
        out = np.empty(len(r) * int(world), dtype=np.float64)
        cd = cfg.descriptor() if cfg is not None else None
        _lib.check(_lib.lib().hcub_worker_exchange_records(self._h, comm, _lib.dptr(r), len(r), int(col_partial),
                                                           int(col_bound), C.byref(cd) if cd is not None else None,
                                                           _lib.dptr(out)))
        return out.tolist()

    def classify_commit(self, global_integral: float, cfg) -> ClassifyResult:
        out = _lib.hcub_classify_out()
        cd = cfg.descriptor()
        _lib.check(_lib.lib().hcub_worker_classify_commit(self._h, float(global_integral), C.byref(cd), C.byref(out)))
        return ClassifyResult(out.finalized_integral, out.finalized_error, int(out.width_guard_hits),
                              int(out.n_finalized), int(out.n_split), out.children_integral, out.children_error,
                              bool(out.split_done))

    def classify_discard(self) -> None:
        _lib.check(_lib.lib().hcub_worker_classify_discard(self._h))

    def evaluate_tail(self, start: int) -> int:
        ev = C.c_int64()
        _lib.check(_lib.lib().hcub_worker_evaluate_tail(self._h, int(start), C.byref(ev)))
        return int(ev.value)

    def reserve(self, rows: int) -> bool:
        """Spare capacity for a split into `rows` children (False: the store's
        fixed capacity does not allow it)."""
        ok = C.c_int32()
        _lib.check(_lib.lib().hcub_worker_reserve(self._h, int(rows), C.byref(ok)))
        return bool(ok.value)

    def classify(self, global_integral: float, cfg) -> ClassifyResult:
        out = _lib.hcub_classify_out()
        cd = cfg.descriptor()
        # split=2: children stay virtual (survivor list) until K1 derives them
        _lib.check(_lib.lib().hcub_worker_classify(self._h, float(global_integral), C.byref(cd), 2, C.byref(out)))
        return ClassifyResult(out.finalized_integral, out.finalized_error, int(out.width_guard_hits),
                              int(out.n_finalized), int(out.n_split), out.children_integral, out.children_error,
                              bool(out.split_done))

    def take_top(self, n: int):
        """Remove the n largest-error rows (numpy stable argsort(-error)
        order) -> (lo, hi, error, integral) host arrays."""
        n = min(int(n), len(self))
        lo = np.empty((n, self.d))
        hi = np.empty((n, self.d))
        E = np.empty(n)
        I = np.empty(n)
        got = C.c_int64()
        if n:
            _lib.check(_lib.lib().hcub_worker_take_top(self._h, n, _lib.dptr(lo), _lib.dptr(hi), _lib.dptr(E),
                                                       _lib.dptr(I), 0, C.byref(got)))
        return lo, hi, E, I

    def take_top_device(self, n: int, lo_ptr: int, hi_ptr: int, err_ptr: int, int_ptr: int) -> int:
        D = _lib._D
        got = C.c_int64()
        _lib.check(_lib.lib().hcub_worker_take_top(self._h, int(n), C.cast(lo_ptr, D), C.cast(hi_ptr, D),
                                                   C.cast(err_ptr, D), C.cast(int_ptr, D), 1, C.byref(got)))
        return int(got.value)

    def exact_partial(self, which: int) -> ExactPartial:
        """carry + sum of the integral (0) / error (1) column, exactly."""
        slots = np.zeros(68, dtype=np.int64)
        sp = (C.c_int32 * 3)()
        _lib.check(_lib.lib().hcub_worker_exact_partial(self._h, which, _lib.iptr(slots),
                                                        C.cast(sp, _lib._I32)))
        v = 0
        for k in range(67, -1, -1):
            v = (v << 32) + int(slots[k])
        return ExactPartial(v, int(sp[0]), int(sp[1]), int(sp[2])) + ExactPartial.of(self.carry[which])

    def timings(self) -> dict:
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        n1, nl = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().hcub_worker_timings(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(n1),
                                                  C.byref(nl)))
        return dict(k1_ms=a.value, k2_ms=b.value, k3_ms=c.value, k1_launches=n1.value, launches=nl.value)
