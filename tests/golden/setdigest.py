"""Order-independent O(n) digest of an active region set (test infrastructure).

Used for the long reference traces (up to ~6e7 regions), where a sha256 over a
lexsorted copy is too slow and too memory-hungry.  Each row (lo_0..lo_{d-1},
hi_0..hi_{d-1}) is hashed from the raw IEEE-754 bit patterns with a
splitmix64-style mixer; the set digest is (count, sum mod 2^64, xor) of the
row hashes, so it does not depend on row order and any changed bit of any
coordinate changes it.  Shared by `make_golden.py` (reference side) and the
GPU parity tests (device side); it is plain numpy, so both sides compute the
same digest bit for bit.
"""
import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(x):
    x = x ^ (x >> np.uint64(30))
    x = x * _M1
    x = x ^ (x >> np.uint64(27))
    x = x * _M2
    return x ^ (x >> np.uint64(31))


def set_digest(lo, hi, chunk=1 << 22):
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    n = lo.shape[0]
    total = np.uint64(0)
    acc_x = np.uint64(0)
    with np.errstate(over="ignore"):
        for s in range(0, n, chunk):
            h = np.full(min(chunk, n - s), _G, dtype=np.uint64)
            for cols in (lo, hi):
                blk = np.ascontiguousarray(cols[s:s + chunk]).view(np.uint64)
                for j in range(blk.shape[1]):
                    h = _mix(h ^ blk[:, j]) + _G
            total = total + np.add.reduce(h, dtype=np.uint64)
            acc_x = acc_x ^ np.bitwise_xor.reduce(h)
    return f"{n}:{int(total):016x}:{int(acc_x):016x}"
