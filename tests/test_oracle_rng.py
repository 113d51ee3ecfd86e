"""Pins for the oracle's random streams and deterministic arithmetic.

Every check compares the oracle with something other than itself: published
known-answer vectors, exact rational arithmetic, closed forms or statistics.
"""
import math
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _anchors():
    out = {}
    for line in open(os.path.join(GOLD, "paper_anchors.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, val = line.split()[:2]
        out[name] = float(val)
    return out


def test_philox_known_answers(ora):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        assert ora.philox(v[0:4], v[4:6]) == tuple(v[6:10])
        n += 1
    assert n == 3


def test_u24_exact_and_symmetric(ora):
    rng = np.random.default_rng(1)
    for w in [0, 1, 255, 256, 0xFFFFFFFF, 0x80000000, *rng.integers(0, 2**32, 200)]:
        u = ora.u24(int(w))
        assert 0.0 < u < 1.0
        assert float(np.float32(u)) == u                   # exactly representable in binary32
        assert Fraction(u) == Fraction(2 * (int(w) >> 9) + 1, 2**24)
        assert ora.u24(int(w) ^ 0xFFFFFFFF) + u == 1.0     # mirror symmetry of the grid


def test_box_muller_statistics(ora):
    """N(0,1): moments and a KS test against the normal CDF (scipy)."""
    from scipy import stats
    rng = np.random.default_rng(2)
    w = rng.integers(0, 2**32, size=(60000, 2), dtype=np.uint64)
    z = np.array([ora.box_muller(int(a), int(b)) for a, b in w]).ravel()
    assert abs(z.mean()) < 4.0 / math.sqrt(z.size)
    assert abs(z.var() - 1.0) < 4.0 * math.sqrt(2.0 / z.size)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    pairs = z.reshape(-1, 2)
    assert abs(np.corrcoef(pairs[:, 0], pairs[:, 1])[0, 1]) < 4.0 / math.sqrt(pairs.shape[0])
    # Box-Muller identity: n0^2 + n1^2 = -2 ln u1
    a, b = 123456789, 987654321
    n0, n1 = ora.box_muller(a, b)
    assert math.isclose(n0 * n0 + n1 * n1, -2.0 * math.log(ora.u24(a)), rel_tol=1e-14)


def test_det_exp2_coefficients_are_rounded_taylor_terms(ora):
    """c_j = RN((ln 2)^j / j!) -- recomputed with 60-digit decimal arithmetic."""
    getcontext().prec = 60
    ln2 = Decimal(2).ln()
    for j, c in enumerate(ora.det_coeffs()):
        exact = ln2 ** j / math.factorial(j)
        # correctly rounded double: the nearest binary64 to the exact value
        f = float(exact)
        cand = [f, math.nextafter(f, math.inf), math.nextafter(f, -math.inf)]
        best = min(cand, key=lambda x: abs(Decimal(x) - exact))
        assert c == best, j


def test_det_exp2_accuracy_and_integers(ora):
    for n in range(-1022, 1000, 37):
        assert ora.det_exp2(float(n)) == 2.0 ** n
    rng = np.random.default_rng(3)
    getcontext().prec = 40
    for y in np.concatenate([rng.uniform(-60, 40, 2000), rng.uniform(-1, 0, 500)]):
        exact = Decimal(2) ** Decimal(float(y))
        got = Decimal(ora.det_exp2(float(y)))
        assert abs(got - exact) / exact < Decimal("5e-16")
    assert ora.det_exp2(-1023.5) == 0.0           # below the normal range by definition (R26)
    assert ora.det_exp2(-math.inf) == 0.0


def test_det_quant_matches_exact_floor(ora):
    """det_quant(d) = floor(2^(32+d)) (Decimal), except within 1e-6 of an integer."""
    getcontext().prec = 50
    assert ora.det_quant(0.0) == 2**32
    assert ora.det_quant(-1.0) == 2**31
    assert ora.det_quant(-32.0) == 1
    assert ora.det_quant(-32.0000001) == 0
    assert ora.det_quant(-math.inf) == 0
    assert ora.det_quant(float("nan")) == 0
    rng = np.random.default_rng(4)
    for d in rng.uniform(-32, 0, 3000):
        exact = Decimal(2) ** Decimal(float(32.0 + d))   # det_quant rounds 32+d first
        fl = int(exact)
        if abs(exact - fl) < Decimal("1e-6") or abs(exact - fl - 1) < Decimal("1e-6"):
            continue
        assert ora.det_quant(float(d)) == fl


def test_sample_schedule_paper_values(ora):
    a = _anchors()
    assert ora.sample_schedule(0) == a["schedule_0"]
    assert ora.sample_schedule(100) == a["schedule_100"]
    assert sum(ora.sample_schedule(j) for j in range(101)) == a["schedule_sum_0_100"]
    seq = [ora.sample_schedule(j) for j in range(101)]
    assert all(b >= x for x, b in zip(seq, seq[1:]))        # monotone (Alg.1 l.2)


def test_stream_tags_are_disjoint(ora):
    """Different tags / indices give different words (no accidental stream reuse)."""
    seen = set()
    for tag in range(1, 9):
        for x0 in range(3):
            seen.add(ora.r64(tag, x0, 1, 0x5EED0001))
    assert len(seen) == 24


def test_paper_weight_sums(ora):
    a = _anchors()
    from paper_1506_02869_b200 import scenarios as sc
    scn = sc.base_scenario()
    assert math.isclose(sum(scn["alpha_dep"]), a["alpha_dep_sum"])
    assert math.isclose(sum(scn["alpha_arr"]), a["alpha_arr_sum"])
    assert scn["A_c"] == a["A_c"]
