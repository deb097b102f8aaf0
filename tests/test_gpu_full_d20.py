"""Full-output parity at the headline size (BASELINE.json config 4, D = 20): every one of the
3^20 = 3,486,784,401 cells against the oracle (Algorithm 1, PAPER.md 40-60), streamed in
contiguous blocks of 3^14 cells through ``oracle.conv_cells`` on all host cores.

* Exp(1)-normalised fp64 (the benchmark inputs): max|z_gpu - z_oracle| <= 1e-12 sum|x| sum|y|
  over all cells (BASELINE.json tolerance), and every cell without a 1-trit bit-exact: such a
  cell is a single product x[i] y[j] (PAPER.md 166-171) that every evaluation point leaves
  alone, so one rounding on both sides.
* Integer-valued fp64 inputs in [0, 15]: the method is exact "when the dynamic range allows
  (a+b)-a = b" (PAPER.md 191-192; Table 1 reports error 0, PAPER.md 307).  Every
  evaluation, product, pair sum and interpolation is an integer below 15^2 4^20 < 2^53, so
  the fp64 path must equal the oracle bit for bit on every cell.  The same inputs as int64
  run the plain int64 engine at the D = 20 geometry (uint64 wrap, R3), also bit-exact.
* All-ones and separable inputs at D = 20 against their closed forms (PAPER.md 168-170;
  axis peeling PAPER.md 153-164) over the whole output, fp64 and int64.

These tests take minutes (the oracle does 4^20 = 1.1e12 pair products per full pass).
"""
import numpy as np
import pytest

import hcgen

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

D = 20
BLOCK = 3 ** 14          # cells per streamed block (one slab of the two-level engine)
M = 3 ** D


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_00206_b200.hc as hcmod
    return hcmod


def _gpu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(hc, x, y):
    z = torch.empty(M, dtype=torch.float64 if x.dtype == np.float64 else torch.int64, device="cuda")
    hc.Plan(D, str(x.dtype)).convolve(_gpu(x), _gpu(y), z)
    torch.cuda.synchronize()
    return z


def _digits_ones(k, ndig):
    c = np.zeros(k.shape, dtype=np.int64)
    k = k.copy()
    for _ in range(ndig):
        c += (k % 3 == 1)
        k //= 3
    return c


_LOW_ONES = None


def _ones_count_block(k0, n):
    """number of 1-trits of every flat index in [k0, k0 + n) (blocks are whole 3^14 slabs:
    low 14 digits from a table, high 6 digits from the block index)."""
    global _LOW_ONES
    if _LOW_ONES is None:
        _LOW_ONES = _digits_ones(np.arange(BLOCK, dtype=np.int64), 14)
    assert k0 % BLOCK == 0 and n == BLOCK
    return _LOW_ONES + int(_digits_ones(np.array([k0 // BLOCK]), D - 14)[0])


def _blocks():
    for k0 in range(0, M, BLOCK):
        yield k0, BLOCK


def test_c4_d20_fp64_every_cell(hc, orc):
    x, y = hcgen.config_inputs("c4_d20_f64")
    z = _run(hc, x, y)
    scale = float(np.abs(x).sum() * np.abs(y).sum())
    worst = 0.0
    for k0, n in _blocks():
        want = orc.conv_cells(x, y, np.arange(k0, k0 + n, dtype=np.uint64))
        got = z[k0:k0 + n].cpu().numpy()
        worst = max(worst, float(np.max(np.abs(got - want))))
        assert worst <= 1e-12 * scale, f"block at {k0}: max err {worst:.3e}"
        single = _ones_count_block(k0, n) == 0
        assert np.array_equal(got[single], want[single]), f"single-product cells differ in block {k0}"
    print(f"D=20 fp64 every cell: max |err| = {worst:.3e} (tolerance {1e-12 * scale:.3e})")


def test_d20_integer_valued_exact_every_cell(hc, orc):
    xi, yi = hcgen.make_pair(D, "int64", "uniform", 2020, 0, 15)
    xf, yf = xi.astype(np.float64), yi.astype(np.float64)
    torch.cuda.empty_cache()
    zf = _run(hc, xf, yf)
    zi = _run(hc, xi, yi)
    for k0, n in _blocks():
        want = orc.conv_cells(xi, yi, np.arange(k0, k0 + n, dtype=np.uint64))
        gi = zi[k0:k0 + n].cpu().numpy()
        assert np.array_equal(gi, want), f"int64 engine differs in block {k0}"
        gf = zf[k0:k0 + n].cpu().numpy()
        assert np.array_equal(gf, want.astype(np.float64)), f"fp64 not exact in block {k0}"


def _separable_part(c, k, axes):
    out = np.ones(k.shape, dtype=np.int64)
    k = k.copy()
    for b in axes:
        out *= c[b][k % 3]
        k //= 3
    return out


@pytest.mark.parametrize("dtype", ["int64", "float64"])
def test_d20_closed_forms_every_cell(hc, dtype):
    # all-ones: z[k] = 2^{#1-trits(k)}; separable: z = (x)_d (x_d * y_d)
    x, y = hcgen.all_ones(D, dtype)
    z = _run(hc, x, y)
    for k0, n in _blocks():
        want = (1 << _ones_count_block(k0, n)).astype(dtype)
        assert np.array_equal(z[k0:k0 + n].cpu().numpy(), want), f"all-ones block {k0}"
    del z
    torch.cuda.empty_cache()
    # int64: factors in {1, 2} (z <= 8^20 < 2^63, uint64 wrap exact); fp64: factors in {0, 1}, so
    # every evaluation-domain value (<= 4^20) and interpolation stays an exact integer < 2^53
    fx, fy = hcgen.separable_factors(D, seed=1120, lo=1 if dtype == "int64" else 0, hi=2 if dtype == "int64" else 1)
    xs, ys = hcgen.tensor_product(fx).astype(dtype), hcgen.tensor_product(fy).astype(dtype)
    z = _run(hc, xs, ys)
    c = [np.array([fx[b, 0] * fy[b, 0], fx[b, 0] * fy[b, 1] + fx[b, 1] * fy[b, 0], fx[b, 1] * fy[b, 1]],
                  dtype=np.int64) for b in range(D)]
    low = _separable_part(c, np.arange(BLOCK, dtype=np.int64), range(14))
    for k0, n in _blocks():
        high = int(_separable_part(c, np.array([k0 // BLOCK]), range(14, D))[0])
        assert np.array_equal(z[k0:k0 + n].cpu().numpy(), (low * high).astype(dtype)), f"separable block {k0}"
    del z
    torch.cuda.empty_cache()
