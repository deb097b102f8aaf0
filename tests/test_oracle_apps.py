"""Pins for the application oracles (oracle/apps.py) against what the paper
and the mathematics fix: hand-derived values (tests/golden/), independent multi-index brute
force, the ordinary 1-D convolution, closed forms and the p-norm bounds.  CPU only."""
import itertools
import os

import numpy as np
import pytest

import hcgen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                key, *vals = line.split()
                out[key] = [int(v) for v in vals]
    return out


@pytest.fixture(scope="module")
def apps(orc):
    import oracle.apps as a
    return a


# ---- f4: differences (PAPER.md 35-38, 147-149) ----------------------------------------
def test_difference_d1_worked(apps):
    g = _golden("difference_d1.txt")
    z = apps.difference_pmf(np.array(g["x"], dtype=np.int64), np.array(g["y"], dtype=np.int64))
    assert z.tolist() == g["z"]


def _difference_bruteforce(x, y, D):
    out = [0] * 3 ** D
    for i in itertools.product((0, 1), repeat=D):
        for j in itertools.product((0, 1), repeat=D):
            d = [a - b for a, b in zip(i, j)]
            fi = sum(v << b for b, v in enumerate(i))
            fj = sum(v << b for b, v in enumerate(j))
            out[sum((v + 1) * 3 ** b for b, v in enumerate(d))] += int(x[fi]) * int(y[fj])
    return out


@pytest.mark.parametrize("D", [1, 2, 3, 4])
def test_difference_bruteforce_and_invariants(apps, D):
    x = hcgen.uniform_int(8100 + D, 0, 1 << D, -20, 20)
    y = hcgen.uniform_int(8100 + D, 1, 1 << D, -20, 20)
    z = apps.difference_pmf(x, y)
    assert z.tolist() == _difference_bruteforce(x, y, D)
    assert int(z.sum()) == int(x.sum()) * int(y.sum())            # mass
    # negation: X - Y = -(Y - X), i.e. trits k_b -> 2 - k_b (reversal of the flat index)
    assert np.array_equal(apps.difference_pmf(y, x), z[::-1])


def test_difference_of_probability_vectors(apps):
    # a PMF: nonnegative, sums to 1, and the mean of d_b is E[X_b] - E[Y_b] on every axis
    D = 6
    x, y = hcgen.make_pair(D, "float64", "exp_norm", 8200)
    z = apps.difference_pmf(x, y)
    assert (z >= 0).all() and abs(z.sum() - 1.0) < 1e-12
    k = np.arange(3 ** D)
    for b in range(D):
        d = (k // 3 ** b) % 3 - 1
        ex = x[(np.arange(1 << D) >> b) & 1 == 1].sum()
        ey = y[(np.arange(1 << D) >> b) & 1 == 1].sum()
        assert abs((d * z).sum() - (ex - ey)) < 1e-12


# ---- f1: carries (PAPER.md 354-373) ---------------------------------------------------
def test_carry_free_worked_example(apps, orc):
    g = _golden("carry_free_7_5.txt")
    D = g["D"][0]
    x = np.zeros(1 << D, dtype=np.int64)
    y = np.zeros(1 << D, dtype=np.int64)
    x[g["i"][0]] = 1
    y[g["j"][0]] = 1
    out = apps.conv1d_carryfree_then_carries(x, y)
    assert np.nonzero(out)[0].tolist() == g["carried"] and out.sum() == 1


@pytest.mark.parametrize("D", [1, 2, 5, 9, 12])
def test_carries_give_ordinary_convolution(apps, D):
    # carry-free convolution followed by the carries is the ordinary 1-D convolution
    x = hcgen.uniform_int(8300 + D, 0, 1 << D, -1000, 1000)
    y = hcgen.uniform_int(8300 + D, 1, 1 << D, -1000, 1000)
    assert np.array_equal(apps.conv1d_carryfree_then_carries(x, y), np.convolve(x, y))


def test_carry_values_bruteforce(apps):
    D = 5
    v = apps.carry_values(D)
    for k in range(3 ** D):
        digits = [(k // 3 ** b) % 3 for b in range(D)]
        assert v[k] == sum(d << b for b, d in enumerate(digits))


# ---- f2: max-convolution (PAPER.md 341-352) -------------------------------------------
def _maxconv_bruteforce(x, y, D):
    out = [None] * 3 ** D
    for i in itertools.product((0, 1), repeat=D):
        for j in itertools.product((0, 1), repeat=D):
            fi = sum(v << b for b, v in enumerate(i))
            fj = sum(v << b for b, v in enumerate(j))
            k = sum((a + b) * 3 ** t for t, (a, b) in enumerate(zip(i, j)))
            v = int(x[fi]) * int(y[fj])
            out[k] = v if out[k] is None else max(out[k], v)
    return out


@pytest.mark.parametrize("D", [1, 2, 3])
def test_maxconv_exact_bruteforce(apps, D):
    x = hcgen.uniform_int(8400 + D, 0, 1 << D, 0, 30)
    y = hcgen.uniform_int(8400 + D, 1, 1 << D, 0, 30)
    assert apps.maxconv_exact(x, y).tolist() == _maxconv_bruteforce(x, y, D)


def test_pnorm_bounds_and_limits(apps, orc):
    D = 8
    x = hcgen.uniform_int(8500, 0, 1 << D, 1, 15).astype(np.float64)
    y = hcgen.uniform_int(8500, 1, 1 << D, 1, 15).astype(np.float64)
    M = apps.maxconv_exact(x, y)
    nk = np.array([2 ** sum(1 for b in range(D) if (k // 3 ** b) % 3 == 1) for k in range(3 ** D)], dtype=np.float64)
    for p in (2.0, 8.0, 64.0):
        E = apps.maxconv_pnorm(x, y, p)
        assert (E >= M * (1 - 1e-12)).all()                      # the p-norm never undercuts the max
        assert (E <= M * nk ** (1.0 / p) * (1 + 1e-12)).all()    # relative error <= 1 - n^(-1/p)
    # p = 1 is the ordinary (sum, x) convolution
    assert np.allclose(apps.maxconv_pnorm(x, y, 1.0), orc.conv(x, y), rtol=1e-12, atol=0)


def test_pnorm_rounding_exact_for_bounded_integers(apps):
    # PAPER.md 346-352: with M (n^(1/p) - 1) < 0.5 on every cell, rounding gives the exact max
    D = 6
    x = hcgen.uniform_int(8600, 0, 1 << D, 0, 3).astype(np.float64)
    y = hcgen.uniform_int(8600, 1, 1 << D, 0, 3).astype(np.float64)
    V2 = 9.0
    p = float(np.ceil(np.log(2.0 ** D) / np.log(1 + 0.5 / V2))) + 1
    assert np.array_equal(np.rint(apps.maxconv_pnorm(x, y, p)), apps.maxconv_exact(x, y))
