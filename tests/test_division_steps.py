"""CPU pin of the standardization's division (csrc/prep.cu div_rn): a / b from rs = RN(1/b) by
q = RN(a rs), r = RN(a - b q) (an fma: exact here), RN(q + r rs) — the final steps of IEEE
division — must equal the correctly rounded a / b.  Exact rational arithmetic stands in for the
device's fma; inputs span the standardization's range (|a / b| up to sqrt(n) and beyond, column
scales over 2^+-40) plus hand-picked hard cases."""
import random
from fractions import Fraction as F

import pytest


def div_steps(a, b):
    rs = 1.0 / b
    q = a * rs
    r = float(F(a) - F(b) * F(q))          # fma(-b, q, a): one rounding
    return float(F(r) * F(rs) + F(q))      # fma(r, rs, q): one rounding


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_division_steps_equal_ieee_division(seed):
    rng = random.Random(seed)
    for _ in range(20000):
        b = rng.uniform(1e-3, 1e3) * 2.0 ** rng.randint(-40, 40)
        a = rng.gauss(0.0, 1.0) * b * rng.choice([1e-6, 0.1, 1.0, 30.0, 1e4])
        assert div_steps(a, b) == a / b, (a, b)


def test_division_steps_hard_cases():
    cases = [(1.0, 3.0), (2.0, 3.0), (-7.0, 7.0), (0.0, 5.0), (1.0, 1.0 + 2.0 ** -52),
             (1.0 - 2.0 ** -53, 1.0 + 2.0 ** -52), (5.0, 0.1), (0.3, 0.1), (1e300, 1e10),
             (3.0, 2.0 ** -30 * 3.0)]
    for a, b in cases:
        assert div_steps(a, b) == a / b, (a, b)
