"""Region geometry semantics (mirrors the reference's pkg/tests/test_regions.py
expectations; host-side bookkeeping)."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2511_01573_b200.regions import HyperRect, RegionStore, split, uniform_partition, volume


def test_volume_and_validation():
    assert volume(HyperRect.unit_cube(3)) == 1.0
    assert volume(HyperRect([0.0, 0.0], [1.0, 0.5])) == 0.5
    assert volume(HyperRect([0.25] * 4, [0.75] * 4)) == 0.0625
    for lo, hi in (([0.0, 1.0], [1.0, 1.0]), ([0.0], [np.inf]), (np.empty(0), np.empty(0))):
        with pytest.raises(ValueError):
            HyperRect(lo, hi)


def test_split():
    a, b = split(HyperRect.unit_cube(2), 0)
    assert a.hi.tolist() == [0.5, 1] and b.lo.tolist() == [0.5, 0]
    a, b = split(HyperRect([0.2, 0.0], [0.6, 1.0]), 0)
    assert b.lo[0] == a.hi[0] == 0.2 + 0.5 * (0.6 - 0.2)
    with pytest.raises(ValueError):
        split(HyperRect.unit_cube(2), 2)


def test_partition_ties_and_octants():
    parts = uniform_partition(HyperRect.unit_cube(2), 2)
    assert parts[0].hi.tolist() == [0.5, 1.0]  # tie -> lowest axis
    parts = uniform_partition(HyperRect.unit_cube(3), 8)
    assert sorted(tuple(p.lo) for p in parts) == sorted(
        (x, y, z) for x in (0, 0.5) for y in (0, 0.5) for z in (0, 0.5))


@settings(max_examples=50, deadline=None)
@given(st.integers(1, 4), st.integers(1, 40))
def test_partition_covers_domain(d, k):
    parts = uniform_partition(HyperRect.unit_cube(d), k)
    assert len(parts) == k
    assert sum(volume(p) for p in parts) == pytest.approx(1.0, rel=1e-14)


def test_store_roundtrip_extract_compact():
    s = RegionStore.from_arrays(np.arange(5)[:, None] * 1.0, np.arange(5)[:, None] + 1.0,
                                integral=np.arange(5) * 1.0)
    b = s.extract([3, 1])
    assert b.lo[:, 0].tolist() == [3.0, 1.0]
    assert s.lo[:, 0].tolist() == [0.0, 2.0, 4.0]
    s.active[1] = False
    s.compact()
    assert s.lo[:, 0].tolist() == [0.0, 4.0]


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 9), st.integers(1, 200), st.integers(0, 2 ** 31))
def test_partition_arrays_match_oracle(d, k, seed):
    """The list-free partition used on every run equals the oracle's restatement
    of ref regions.py:92-111 bit for bit (ragged domains, ties)."""
    from oracle import hcub_oracle as orc
    from paper_2511_01573_b200.regions import partition_arrays
    rng = np.random.default_rng(seed)
    lo = rng.standard_normal(d) * rng.choice([1e-3, 1.0, 1e3])
    hi = lo + rng.choice([1.0, 2.0, 0.1]) * (1 + rng.integers(0, 3, size=d))
    a, b = partition_arrays(HyperRect(lo, hi), k)
    ea, eb = orc.partition(lo, hi, k)
    assert np.array_equal(a, ea) and np.array_equal(b, eb)
