"""The device superaccumulator (K2/K3 global sums) must equal math.fsum bit
for bit - the reference's exact_sum_with (ref driver.py:43-50)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def cases():
    rng = np.random.default_rng(7)
    yield [0.1] * 10, 0.0
    yield [1e100, 1.0, -1e100], 0.0
    yield [2.0 ** -1074] * 3 + [2.0 ** -1022], 0.0
    yield [1.0, 2.0 ** -53], 0.0                       # tie -> even
    yield [1.0, 2.0 ** -53, 2.0 ** -105], 0.0          # tie broken by sticky
    yield [1.0 + 2.0 ** -52, 2.0 ** -53], 0.0          # tie -> round up to even
    yield [-5.5, 5.5, -0.0], 0.0
    yield [], 3.25
    yield [1.7976931348623157e308, -1.7976931348623157e308, 1.0], 0.5
    for _ in range(30):
        n = int(rng.integers(1, 5000))
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
        yield x.tolist(), float(rng.standard_normal() * 1e10)
    for _ in range(10):
        x = rng.random(20000) * 1e17
        x = np.concatenate([x, -x[: 10000] * (1 + 1e-16)])
        yield x.tolist(), 0.0


@pytest.mark.parametrize("i_case", range(49))
def test_device_fsum_bit_exact(i_case):
    from paper_2511_01573_b200.driver import device_exact_sum
    x, carry = list(cases())[i_case]
    want = math.fsum([carry, *x])
    got = device_exact_sum(x, carry)
    assert got == want or (math.isnan(got) and math.isnan(want)), (got, want)
    assert math.copysign(1, got) == math.copysign(1, want) or got != 0


def test_device_fsum_specials():
    from paper_2511_01573_b200.driver import device_exact_sum
    assert device_exact_sum([1.0, math.inf]) == math.inf
    assert device_exact_sum([1.0, -math.inf]) == -math.inf
    assert math.isnan(device_exact_sum([math.inf, -math.inf]))
    assert math.isnan(device_exact_sum([1.0, math.nan]))
