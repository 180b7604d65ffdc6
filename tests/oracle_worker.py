"""Test double for DeviceWorker backed by the CPU oracle (tests only).

Lets the distributed engine's host protocol (paper_2511_01573_b200/distributed.py)
run on machines without a GPU - in-process and over gloo process groups - and
be checked against the reference's own logs.  Never used by the product path.
"""
from fractions import Fraction

import numpy as np

from oracle import hcub_oracle as orc
from paper_2511_01573_b200.worker import ClassifyResult, ExactPartial, SCALE_BITS


class OracleWorker:
    def __init__(self, f, d, dlo, dhi):
        self.f = f
        self.d = d
        self.dlo = np.asarray(dlo, dtype=float)
        self.dhi = np.asarray(dhi, dtype=float)
        self.tab = orc.gm_table(d)
        self.K = self.tab.K
        self.store = orc.Store(np.zeros((0, d)), np.zeros((0, d)))
        self.fin = (0.0, 0.0)

    def __len__(self):
        return len(self.store)

    def append(self, lo, hi, integral=None, error=None):
        lo = np.atleast_2d(np.asarray(lo, dtype=float))
        hi = np.atleast_2d(np.asarray(hi, dtype=float))
        m = lo.shape[0]
        s = self.store
        s.lo = np.concatenate([s.lo, lo]); s.hi = np.concatenate([s.hi, hi])
        s.I = np.concatenate([s.I, np.zeros(m) if integral is None else integral])
        s.E = np.concatenate([s.E, np.zeros(m) if error is None else error])
        s.axis = np.concatenate([s.axis, np.full(m, -1, dtype=np.int64)])

    @property
    def carry(self):
        return self.fin

    @carry.setter
    def carry(self, v):
        self.fin = (float(v[0]), float(v[1]))

    def evaluate(self):
        pi, pe = orc.evaluate(self.store, self.tab, self.f, self.fin)
        return pi, pe, len(self.store) * self.K

    def evaluate_tail(self, start):
        s = self.store
        if start >= len(s):
            return 0
        I, E, S, ev = orc.eval_regions(self.tab, s.lo[start:], s.hi[start:], self.f)
        s.I[start:], s.E[start:], s.axis[start:] = I, E, np.argmax(S, axis=1)
        return ev

    def classify(self, gI, cfg):
        kids, fin, wall, nf, ns = orc.classify_split(self.store, gI, self.fin, cfg.tau_rel, self.dlo, self.dhi,
                                                     cfg.abs_floor, cfg.classifier.safety, cfg.min_width_ulp_factor)
        self.store, self.fin = kids, fin
        return ClassifyResult(fin[0], fin[1], wall, nf, ns, float(np.sum(kids.I)), float(np.sum(kids.E)), True)

    def take_top(self, n):
        b = orc.take_top(self.store, n)
        return b.lo, b.hi, b.E, b.I

    def read(self):
        s = self.store
        return s.lo, s.hi, s.I, s.E, s.axis

    def exact_partial(self, which):
        vals = (self.store.I if which == 0 else self.store.E).tolist() + [self.fin[which]]
        acc = ExactPartial(0)
        for v in vals:
            acc = acc + ExactPartial.of(v)
        return acc

    def close(self):
        pass


class OverlapOracleWorker(OracleWorker):
    """Adds the device worker's split evaluation (hcub_worker_evaluate_begin /
    _end): rows present at begin are evaluated there, rows appended before end
    are evaluated at end, and the partials cover every row - so the engine's
    overlapped delivery order runs on CPU too."""

    def evaluate_begin(self):
        s = self.store
        self._n0 = len(s)
        if self._n0:
            I, E, S, _ = orc.eval_regions(self.tab, s.lo, s.hi, self.f)
            s.I[:self._n0], s.E[:self._n0], s.axis[:self._n0] = I, E, np.argmax(S, axis=1)

    def evaluate_end(self):
        self.evaluate_tail(self._n0)
        s = self.store
        return orc.fsum_with(self.fin[0], s.I), orc.fsum_with(self.fin[1], s.E), len(s) * self.K


def factory(spec, dlo, dhi, overlap=False):
    from conftest import oracle_f
    f = oracle_f(spec)
    cls = OverlapOracleWorker if overlap else OracleWorker
    return lambda rank: cls(f, spec["d"], dlo, dhi)
