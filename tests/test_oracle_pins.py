"""Pins for the oracle (oracle/hc_oracle.c) against what the paper and the mathematics fix.

Each test names the passage it follows.  None of them re-types the oracle's own loop: they
use hand-derived values (tests/golden/), closed forms, invariants, an independent
multi-index brute force, exact rational arithmetic and a generating-function identity.
CPU only (no `gpu` marker).
"""
from fractions import Fraction
import itertools
import os

import numpy as np
import pytest

import hcgen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            out[key] = [int(v) for v in vals]
    return out


# ---------------------------------------------------------------------------------------
# Independent multi-index brute force (PAPER.md 40-60, Algorithm 1 with vector indices).
# Indices are D-tuples; flattening is written separately from the oracle: input
# weight 2^b, output weight 3^b for axis b (reading R1).
def brute_force(x, y, D):
    z = {}
    for i in itertools.product((0, 1), repeat=D):
        for j in itertools.product((0, 1), repeat=D):
            k = tuple(a + b for a, b in zip(i, j))
            fi = sum(bit << b for b, bit in enumerate(i))
            fj = sum(bit << b for b, bit in enumerate(j))
            z[k] = z.get(k, 0) + int(x[fi]) * int(y[fj])
    out = [0] * 3 ** D
    for k, v in z.items():
        out[sum(d * 3 ** b for b, d in enumerate(k))] = v
    return out


@pytest.mark.parametrize("D", [1, 2, 3, 4])
def test_bruteforce_multiindex(orc, D):
    for seed in range(3):
        x = hcgen.uniform_int(7000 + seed, 0, 1 << D, -50, 50)
        y = hcgen.uniform_int(7000 + seed, 1, 1 << D, -50, 50)
        want = brute_force(x, y, D)
        assert orc.conv(x, y).tolist() == want
        assert orc.conv_scatter(x, y).tolist() == want
        # fp64 on small integers is exact (every partial sum < 2^53)
        assert orc.conv(x.astype(np.float64), y.astype(np.float64)).tolist() == [float(v) for v in want]


def test_d1_form_golden(orc):
    g = _read_golden("d1_form.txt")
    x = np.array(g["x"], dtype=np.int64)
    y = np.array(g["y"], dtype=np.int64)
    assert orc.conv(x, y).tolist() == g["z"]
    assert orc.conv_scatter(x, y).tolist() == g["z"]


def test_d1_form_symbolic(orc):
    # [a0 b0, a0 b1 + a1 b0, a1 b1]  (PAPER.md 174-176, 259-261)
    for s in range(20):
        a = hcgen.uniform_int(11 + s, 0, 2, -1000, 1000)
        b = hcgen.uniform_int(11 + s, 1, 2, -1000, 1000)
        want = [a[0] * b[0], a[0] * b[1] + a[1] * b[0], a[1] * b[1]]
        assert orc.conv(a, b).tolist() == want


def test_d2_worked_example(orc):
    g = _read_golden("d2_worked_example.txt")
    x = np.array(g["x"], dtype=np.int64)
    y = np.array(g["y"], dtype=np.int64)
    assert orc.conv(x, y).tolist() == g["z"]
    assert orc.conv(x.astype(float), y.astype(float)).tolist() == [float(v) for v in g["z"]]


def test_carry_free_example(orc):
    # PAPER.md 359-365: (1,1,1) + (1,0,1) -> (2,1,2), i.e. 12 after carries
    g = _read_golden("carry_free_7_5.txt")
    D = g["D"][0]
    x = np.zeros(1 << D, dtype=np.int64)
    y = np.zeros(1 << D, dtype=np.int64)
    x[g["i"][0]] = 1
    y[g["j"][0]] = 1
    z = orc.conv(x, y)
    assert z.sum() == 1 and z[g["k_flat"][0]] == 1
    k = g["k_flat"][0]
    digits = [(k // 3 ** b) % 3 for b in range(D)]
    assert digits[::-1] == g["k_digits"]
    assert sum(d << b for b, d in enumerate(digits)) == g["carried"][0] == 7 + 5


def _ones_trits(k, D):
    return sum(1 for b in range(D) if (k // 3 ** b) % 3 == 1)


@pytest.mark.parametrize("D", [1, 3, 5, 8, 11])
def test_all_ones_closed_form(orc, D):
    # x = y = 1: z[k] = number of (i,j) with i+j=k = 2^{#trits equal to 1}
    # (PAPER.md 168-170: k_1 = 1 has two (i_1, j_1) cases, 0 and 2 have one)
    x, y = hcgen.all_ones(D)
    z = orc.conv(x, y)
    want = np.array([2 ** _ones_trits(k, D) for k in range(3 ** D)], dtype=np.int64)
    assert np.array_equal(z, want)
    zf = orc.conv(x.astype(float), y.astype(float))
    assert np.array_equal(zf, want.astype(float))


def _separable_expected(fx, fy):
    # z = tensor product over axes of the 1-D length-2 convolutions (x_d * y_d)
    # (axis peeling, PAPER.md 153-164).  Axis b is the 3^b digit.
    z = np.ones(1, dtype=object)
    for b in range(fx.shape[0]):
        a0, a1 = int(fx[b, 0]), int(fx[b, 1])
        b0, b1 = int(fy[b, 0]), int(fy[b, 1])
        c = [a0 * b0, a0 * b1 + a1 * b0, a1 * b1]
        z = np.concatenate([z * c[0], z * c[1], z * c[2]])
    return z


@pytest.mark.parametrize("D", [2, 6, 10])
def test_separable(orc, D):
    fx, fy = hcgen.separable_factors(D, seed=1103 + D, lo=-3, hi=3)
    x = hcgen.tensor_product(fx)
    y = hcgen.tensor_product(fy)
    want = _separable_expected(fx, fy)
    z = orc.conv(x, y)
    assert [int(v) for v in z] == [int(v) for v in want]


@pytest.mark.parametrize("D", [3, 7])
def test_delta_shift(orc, D):
    # x = delta_a: z[T(a) + T(j)] = y[j], zero elsewhere (SPEC.md 143; PAPER.md 30-34)
    y = hcgen.uniform_int(31, 1, 1 << D, 1, 100)
    for a in [0, 1, (1 << D) - 1, 5 % (1 << D)]:
        x = np.zeros(1 << D, dtype=np.int64)
        x[a] = 1
        z = orc.conv(x, y)
        want = np.zeros(3 ** D, dtype=np.int64)
        ta = sum(((a >> b) & 1) * 3 ** b for b in range(D))
        for j in range(1 << D):
            tj = sum(((j >> b) & 1) * 3 ** b for b in range(D))
            want[ta + tj] = y[j]
        assert np.array_equal(z, want)


@pytest.mark.parametrize("D", [4, 9, 12])
def test_mass_conservation(orc, D):
    x, y = hcgen.make_pair(D, "int64", "uniform", 900 + D, 0, 1000)
    z = orc.conv(x, y)
    assert int(z.sum()) == int(x.sum()) * int(y.sum())


P61 = (1 << 61) - 1


@pytest.mark.parametrize("D", [5, 11])
def test_generating_function_mod_p(orc, D):
    # Algorithm 1 is multiplication of multilinear polynomials:
    #   sum_k z[k] prod_b w_b^{k_b} = P_x(w) P_y(w),  P_x(w) = sum_i x[i] prod_b w_b^{i_b}
    # checked mod p = 2^61 - 1 at random w (Schwartz-Zippel).
    x, y = hcgen.make_pair(D, "int64", "uniform", 4242 + D, 0, 1 << 16)
    z = orc.conv(x, y)
    rng = np.random.default_rng(D)
    for _ in range(3):
        w = [int(v) for v in rng.integers(2, P61, size=D)]
        wz = np.ones(1, dtype=object)
        wx = np.ones(1, dtype=object)
        for b in range(D):
            wz = np.concatenate([wz, wz * w[b] % P61, wz * (w[b] * w[b] % P61) % P61])
            wx = np.concatenate([wx, wx * w[b] % P61])
        lhs = int(sum(int(a) * int(c) % P61 for a, c in zip(z.tolist(), wz.tolist()))) % P61
        px = sum(int(a) * int(c) for a, c in zip(x.tolist(), wx.tolist())) % P61
        py = sum(int(a) * int(c) for a, c in zip(y.tolist(), wx.tolist())) % P61
        assert lhs == px * py % P61


def test_scatter_equals_gather_bitwise(orc):
    # gather visits each cell's pairs in Algorithm 1's order, so fp64 results are equal
    for D in (6, 10):
        x, y = hcgen.make_pair(D, "float64", "uniform01", 77 + D)
        assert np.array_equal(orc.conv_scatter(x, y), orc.conv(x, y))


def test_commutativity_and_pow2_scaling(orc):
    D = 9
    x, y = hcgen.make_pair(D, "int64", "uniform", 5, -100, 100)
    assert np.array_equal(orc.conv(x, y), orc.conv(y, x))
    xf, yf = hcgen.make_pair(D, "float64", "exp_norm", 6)
    assert np.array_equal(orc.conv(2.0 * xf, yf), 2.0 * orc.conv(xf, yf))


def test_table1_probe(orc):
    # PAPER.md 322-326: x.flat = y.flat = [1..2^D] -> z[(0,...,0)] = 1 exactly
    D = 11
    x = np.arange(1, (1 << D) + 1, dtype=np.float64)
    z = orc.conv(x, x)
    assert z[0] == 1.0
    assert z[-1] == float((1 << D) ** 2)


def test_int64_wraparound_exact_mod_2_64(orc):
    # DESIGN.md R3: int64 is computed mod 2^64; compare with exact integers reduced mod 2^64
    D = 4
    x = hcgen.uniform_int(3, 0, 1 << D, -(1 << 40), 1 << 40)
    y = hcgen.uniform_int(3, 1, 1 << D, -(1 << 40), 1 << 40)
    exact = brute_force(x, y, D)
    got = orc.conv(x, y)
    for g, e in zip(got.tolist(), exact):
        assert (g - e) % (1 << 64) == 0


def test_fp64_within_rounding_bound_of_exact(orc):
    # fp64 oracle vs exact rational result: each cell is a sum of P = 2^{#1-trits}
    # products, so |err| <= (P+1) u sum|x_i y_j| (standard summation bound, u = 2^-53).
    D = 6
    x, y = hcgen.make_pair(D, "float64", "exp_norm", 1004)
    z = orc.conv(x, y)
    xq = [Fraction(v) for v in x.tolist()]
    yq = [Fraction(v) for v in y.tolist()]
    u = 2.0 ** -53
    for k in range(3 ** D):
        digits = [(k // 3 ** b) % 3 for b in range(D)]
        terms = []
        for i in range(1 << D):
            ib = [(i >> b) & 1 for b in range(D)]
            jb = [d - a for d, a in zip(digits, ib)]
            if all(v in (0, 1) for v in jb):
                j = sum(v << b for b, v in enumerate(jb))
                terms.append(xq[i] * yq[j])
        exact = sum(terms, Fraction(0))
        P = len(terms)
        assert P == 2 ** digits.count(1)
        bound = (P + 1) * u * float(sum(terms, Fraction(0)))
        assert abs(Fraction(z[k]) - exact) <= Fraction(bound) * 1.0001


def test_cells_and_batched_match_full(orc):
    D = 8
    x, y = hcgen.make_pair(D, "float64", "exp_norm", 12)
    z = orc.conv(x, y)
    ks = np.array([0, 1, 2, 100, 3 ** D - 1, 3 ** D // 2], dtype=np.uint64)
    assert np.array_equal(orc.conv_cells(x, y, ks), z[ks.astype(np.int64)])
    xb, yb = hcgen.make_batched_fast(3, D, 0, 255, 1002)
    zb = orc.conv_batched(xb, yb)
    for b in range(3):
        assert np.array_equal(zb[b], orc.conv(xb[b], yb[b]))
    bs = np.array([0, 2, 1], dtype=np.uint64)
    kk = np.array([5, 6560, 0], dtype=np.uint64)
    got = orc.conv_batched_cells_i64(xb, yb, bs, kk)
    assert got.tolist() == [int(zb[int(b), int(k)]) for b, k in zip(bs, kk)]


def test_ternary_map(orc):
    # T(i) = sum_b bit_b(i) 3^b (PAPER.md 109-112)
    for i in [0, 1, 2, 3, 7, 5, (1 << 22) - 1]:
        assert orc.ternary_of_binary(i) == sum(((i >> b) & 1) * 3 ** b for b in range(23))


def test_spec_worked_values_and_zero(orc):
    # SPEC.md 183-184 worked values (golden file, with citations) and the zero annihilator
    # (SPEC.md 138): x * 0 = 0 for any x
    g = _read_golden("spec_examples.txt")
    for n in ("1", "2"):
        x = np.array(g["x" + n], dtype=np.int64)
        y = np.array(g["y" + n], dtype=np.int64)
        assert orc.conv(x, y).tolist() == g["z" + n]
        assert orc.conv(y, x).tolist() == g["z" + n]
    rng = np.random.default_rng(138)
    for D in (1, 3, 6):
        x = rng.integers(-1000, 1000, 1 << D).astype(np.int64)
        assert not orc.conv(x, np.zeros_like(x)).any()


# ---------------------------------------------------------------------------------------
# Direct pins for the two oracle entry points the GPU tests use as checkers beyond the
# full-output gather (orc_conv_batched_f64, orc_conv_cells_i64).  Both are pinned against
# the independent multi-index brute force (PAPER.md 40-60), the all-ones closed form
# (PAPER.md 168-170: z[k] = 2^{#trits(k)=1}) and separable inputs (axis peeling, PAPER.md
# 153-164), never against the oracle's own full-output function.
def _ones_closed_form(D):
    ones = np.zeros(1, dtype=np.int64)
    for _ in range(D):
        ones = np.concatenate([ones, ones + 1, ones])
    return (1 << ones).astype(np.int64)


def _separable_closed_form(fx, fy):
    D = fx.shape[0]
    want = np.ones(1, dtype=np.int64)
    for b in range(D):
        c = [fx[b, 0] * fy[b, 0], fx[b, 0] * fy[b, 1] + fx[b, 1] * fy[b, 0], fx[b, 1] * fy[b, 1]]
        want = np.concatenate([want * c[0], want * c[1], want * c[2]])
    return want


@pytest.mark.parametrize("D", [1, 2, 3, 4])
def test_batched_f64_bruteforce_and_stride(orc, D):
    # every batch row against the brute force of that row (small integers: fp64 exact), in a
    # batch whose rows differ, so a wrong batch stride or row mix-up changes the result
    B = 5
    x = np.stack([hcgen.uniform_int(8100 + b, 0, 1 << D, -40, 40) for b in range(B)]).astype(np.float64)
    y = np.stack([hcgen.uniform_int(8100 + b, 1, 1 << D, -40, 40) for b in range(B)]).astype(np.float64)
    z = orc.conv_batched(x, y)
    assert z.shape == (B, 3 ** D)
    for b in range(B):
        want = brute_force(x[b].astype(np.int64), y[b].astype(np.int64), D)
        assert z[b].tolist() == [float(v) for v in want], f"batch row {b}"


def test_batched_f64_closed_forms(orc):
    # row b: x = c_b * ones, y = d_b * ones -> z = c_b d_b 2^{#1}; row-specific scales pin the
    # batch stride; powers of two keep every product and sum exact in fp64
    D, B = 7, 4
    scale_x = np.array([1.0, 2.0, 0.5, 4.0])
    scale_y = np.array([1.0, 0.25, 8.0, 2.0])
    x = scale_x[:, None] * np.ones((B, 1 << D))
    y = scale_y[:, None] * np.ones((B, 1 << D))
    z = orc.conv_batched(x, y)
    base = _ones_closed_form(D).astype(np.float64)
    for b in range(B):
        assert np.array_equal(z[b], scale_x[b] * scale_y[b] * base)
    # separable rows (integer factors in {1,2}: z <= 8^D exact in fp64 for D = 7)
    fx, fy = hcgen.separable_factors(D, seed=1107, lo=1, hi=2)
    xs = hcgen.tensor_product(fx).astype(np.float64)
    ys = hcgen.tensor_product(fy).astype(np.float64)
    zs = orc.conv_batched(np.stack([xs, ys]), np.stack([ys, xs]))
    want = _separable_closed_form(fx, fy).astype(np.float64)
    assert np.array_equal(zs[0], want) and np.array_equal(zs[1], want)  # commutativity across rows


@pytest.mark.parametrize("D", [2, 3, 4])
def test_cells_i64_bruteforce(orc, D):
    # arbitrary cell order with repeats, out-of-order and the last cell, against the brute force
    x = hcgen.uniform_int(8200 + D, 0, 1 << D, -(1 << 30), 1 << 30)
    y = hcgen.uniform_int(8200 + D, 1, 1 << D, -(1 << 30), 1 << 30)
    want = brute_force(x, y, D)
    rng = np.random.default_rng(D)
    ks = np.concatenate([rng.permutation(3 ** D), [3 ** D - 1, 0, 3 ** D - 1]]).astype(np.uint64)
    got = orc.conv_cells(x, y, ks)
    assert got.dtype == np.int64
    for g, k in zip(got.tolist(), ks.tolist()):
        e = want[int(k)]
        assert (g - e) % (1 << 64) == 0 and g == ((e + (1 << 63)) % (1 << 64)) - (1 << 63)


def test_cells_i64_closed_forms_large_D(orc):
    # D = 18: sampled cells against the all-ones and separable closed forms (exact int64)
    D = 18
    rng = np.random.default_rng(18)
    ks = rng.integers(0, 3 ** D, 4000, dtype=np.uint64)
    ks[:3] = [0, 3 ** D - 1, (3 ** D - 1) // 2]          # corners and the all-ones-trit cell
    x, y = hcgen.all_ones(D)
    assert np.array_equal(orc.conv_cells(x, y, ks), _ones_closed_form(D)[ks.astype(np.int64)])
    fx, fy = hcgen.separable_factors(D, seed=1118, lo=1, hi=2)
    xs, ys = hcgen.tensor_product(fx), hcgen.tensor_product(fy)
    want = _separable_closed_form(fx, fy)
    assert np.array_equal(orc.conv_cells(xs, ys, ks), want[ks.astype(np.int64)])
