"""Parity of the CUDA path (through the C ABI) against the oracle (Algorithm 1, PAPER.md 40-60).

int64: bit-exact at every compared cell.  fp64: max|z_gpu - z_oracle| <= 1e-12 * sum|x| *
sum|y| (BASELINE.json north_star tolerance).  Sizes span several tiles and
ragged tails; BASELINE.json's full sizes are checked in full where the oracle can finish
in seconds (C1, C2, C3) and on sampled cells plus whole-output invariants otherwise (C4).
"""
import numpy as np
import pytest

import hcgen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_00206_b200.hc as hcmod
    return hcmod


def _gpu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(hc, x, y):
    D = x.shape[0].bit_length() - 1
    z = torch.empty(3 ** D, dtype=torch.float64 if x.dtype == np.float64 else torch.int64, device="cuda")
    hc.Plan(D, str(x.dtype)).convolve(_gpu(x), _gpu(y), z)
    torch.cuda.synchronize()
    return z


def _assert_close(got, want, x, y):
    if want.dtype == np.int64:
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, f"{bad.size} int64 cells differ, first at {bad[:5]}: {got[bad[:5]]} vs {want[bad[:5]]}"
    else:
        scale = float(np.abs(x).sum() * np.abs(y).sum())
        err = float(np.max(np.abs(got - want))) if got.size else 0.0
        assert err <= TOL * scale, f"max err {err:.3e} > {TOL} * {scale:.3e}"


@pytest.mark.parametrize("dtype", ["int64", "float64"])
@pytest.mark.parametrize("D", list(range(1, 13)))
def test_single_pair_all_D(hc, orc, D, dtype):
    for seed in (1, 2):
        if dtype == "int64":
            x, y = hcgen.make_pair(D, "int64", "uniform", 100 * D + seed, -1000, 1000)
        else:
            x, y = hcgen.make_pair(D, "float64", "exp_norm", 100 * D + seed)
        got = _run(hc, x, y).cpu().numpy()
        _assert_close(got, orc.conv(x, y), x, y)


@pytest.mark.parametrize("D", [1, 2, 3, 5, 7, 8, 9, 10])
def test_batched_small(hc, orc, D):
    B = 7
    xb, yb = hcgen.make_batched_fast(B, D, 0, 255, 31 + D)
    z = torch.empty((B, 3 ** D), dtype=torch.int64, device="cuda")
    hc.convolve_batched(_gpu(xb), _gpu(yb), z)
    torch.cuda.synchronize()
    assert np.array_equal(z.cpu().numpy(), orc.conv_batched(xb, yb))
    xf = (xb.astype(np.float64) + 0.25) / 256.0
    yf = (yb.astype(np.float64) + 0.5) / 256.0
    zf = torch.empty((B, 3 ** D), dtype=torch.float64, device="cuda")
    hc.convolve_batched(_gpu(xf), _gpu(yf), zf)
    torch.cuda.synchronize()
    want = orc.conv_batched(xf, yf)
    for b in range(B):
        _assert_close(zf[b].cpu().numpy(), want[b], xf[b], yf[b])


def test_config_c1_d10_int64(hc, orc):
    x, y = hcgen.config_inputs("c1_d10_i64")
    got = _run(hc, x, y).cpu().numpy()
    assert np.array_equal(got, orc.conv(x, y))


def test_config_c2_batched_d8_full(hc, orc):
    # BASELINE.json config 2 at full size, every cell of every cube
    x, y = hcgen.config_inputs("c2_b65536_d8_i64")
    B = x.shape[0]
    z = torch.empty((B, 3 ** 8), dtype=torch.int64, device="cuda")
    hc.convolve_batched(_gpu(x), _gpu(y), z)
    torch.cuda.synchronize()
    assert np.array_equal(z.cpu().numpy(), orc.conv_batched(x, y))


@pytest.mark.parametrize("B", [1, 7, 1500])
def test_batched_d8_narrow_ring_boundary(hc, orc, B):
    # batched D = 8 int64 runs in the 32-bit ring when 2^8 max|x| max|y| < 2^31 (every output is
    # a sum of at most 2^8 products, PAPER.md 166-171; ring homomorphism, R3) and in
    # the 64-bit engine otherwise.  Cubes straddle the bound: constant cubes x = a, y = b put
    # 2^8 a b at the all-1 cell, so a b = 2^23 - 1 is the largest safe product (z = 2^31 - 256)
    # and a b = 2^23 the first unsafe one (z = 2^31 needs 64 bits); signs flip the extremes to
    # -2^31 + 256 and -2^31; random cubes mix safe small entries with full-range ones.
    rng = np.random.default_rng(880 + B)
    xb = np.empty((B, 256), dtype=np.int64)
    yb = np.empty((B, 256), dtype=np.int64)
    kinds = rng.integers(0, 6, B)
    for i, k in enumerate(kinds):
        if k == 0:   # largest safe constant cube
            xb[i], yb[i] = 8191, 1025          # 8191 * 1025 = 2^23 - 1
        elif k == 1:  # smallest unsafe constant cube
            xb[i], yb[i] = -2048, 4096          # 2^23, negative: z = -2^31 at the all-1 cell
        elif k == 2:
            xb[i] = rng.integers(-255, 256, 256)
            yb[i] = rng.integers(-255, 256, 256)
        elif k == 3:  # one outlier entry makes the cube unsafe
            xb[i] = rng.integers(0, 256, 256)
            yb[i] = rng.integers(0, 256, 256)
            yb[i, rng.integers(0, 256)] = 1 << 40
        elif k == 4:
            xb[i] = hcgen.splitmix64(9000 + i, 0, 256).view(np.int64)
            yb[i] = hcgen.splitmix64(9000 + i, 1, 256).view(np.int64)
        else:         # INT64_MIN: |x| = 2^63 must not wrap to a small magnitude
            xb[i] = 0
            xb[i, 5] = np.iinfo(np.int64).min
            yb[i] = 1
    if B == 1:
        xb[0], yb[0] = 8191, -1025
    z = torch.empty((B, 3 ** 8), dtype=torch.int64, device="cuda")
    hc.convolve_batched(_gpu(xb), _gpu(yb), z)
    torch.cuda.synchronize()
    assert np.array_equal(z.cpu().numpy(), orc.conv_batched(xb, yb))


def test_batched_d8_concurrent_streams(hc, orc):
    # the 32-bit path's fallback list is per-call stream-ordered scratch: two batches with
    # different unsafe cubes, launched back to back on two streams, must not see each other's list
    B = 600
    xa, ya = hcgen.make_batched_fast(B, 8, 0, 255, 4101)
    xb, yb = hcgen.make_batched_fast(B, 8, 0, 255, 4102)
    xa[::7, 3] = 1 << 36     # every 7th cube of batch a needs 64-bit words
    yb[5::11, 200] = -(1 << 35)
    ga, gb = [(_gpu(x), _gpu(y)) for x, y in ((xa, ya), (xb, yb))]
    za = torch.empty((B, 3 ** 8), dtype=torch.int64, device="cuda")
    zb = torch.empty_like(za)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            hc.convolve_batched(ga[0], ga[1], za, stream=s1)
        with torch.cuda.stream(s2):
            hc.convolve_batched(gb[0], gb[1], zb, stream=s2)
    torch.cuda.synchronize()
    assert np.array_equal(za.cpu().numpy(), orc.conv_batched(xa, ya))
    assert np.array_equal(zb.cpu().numpy(), orc.conv_batched(xb, yb))


def test_config_c3_d16_int64_full(hc, orc):
    x, y = hcgen.config_inputs("c3_d16_i64")
    got = _run(hc, x, y).cpu().numpy()
    assert np.array_equal(got, orc.conv(x, y))


def test_d16_all_ones_and_separable(hc):
    D = 16
    x, y = hcgen.all_ones(D)
    got = _run(hc, x, y).cpu().numpy()
    # closed form z[k] = 2^{#trits(k) == 1}
    ones = np.zeros(1, dtype=np.int64)
    for _ in range(D):
        ones = np.concatenate([ones, ones + 1, ones])
    assert np.array_equal(got, (1 << ones).astype(np.int64))
    fx, fy = hcgen.separable_factors(D, seed=1103, lo=1, hi=2)
    x = hcgen.tensor_product(fx)
    y = hcgen.tensor_product(fy)
    want = np.ones(1, dtype=np.int64)
    for b in range(D):
        c = np.array([fx[b, 0] * fy[b, 0], fx[b, 0] * fy[b, 1] + fx[b, 1] * fy[b, 0], fx[b, 1] * fy[b, 1]])
        want = np.concatenate([want * c[0], want * c[1], want * c[2]])
    assert np.array_equal(_run(hc, x, y).cpu().numpy(), want)


def _sample_cells(D, n, seed):
    m = 3 ** D
    rng = np.random.default_rng(seed)
    ks = rng.integers(0, m, size=n, dtype=np.int64)
    # plus whole contiguous blocks: the first tiles, a ragged tail, and the all-ones-trit region
    ones_idx = sum(3 ** b for b in range(D))
    blocks = [np.arange(0, 3 ** 9), np.arange(m - 3 ** 8 - 17, m),
              np.arange(max(0, ones_idx - 3 ** 8), min(m, ones_idx + 3 ** 8))]
    return np.unique(np.concatenate([ks] + blocks)).astype(np.int64)


@pytest.mark.slow
def test_config_c4_d20_fp64_sampled(hc, orc):
    x, y = hcgen.config_inputs("c4_d20_f64")
    D = 20
    z = _run(hc, x, y)
    ks = _sample_cells(D, 20000, 4)
    got = z[torch.from_numpy(ks).cuda()].cpu().numpy()
    want = orc.conv_cells(x, y, ks.astype(np.uint64))
    _assert_close(got, want, x, y)
    # whole-output invariant: mass conservation sum z = sum x * sum y
    tot = float(z.sum().item())
    assert abs(tot - float(x.sum()) * float(y.sum())) <= 1e-9
    # determinism: a second run is bit-identical
    z2 = _run(hc, x, y)
    assert torch.equal(z, z2)


@pytest.mark.parametrize("ngpu", [2, 3, 8])
def test_sharded_concat_equals_full(hc, ngpu):
    D = 12
    x, y = hcgen.make_pair(D, "int64", "uniform", 55, 0, 1 << 16)
    full = _run(hc, x, y)
    xs, ys = _gpu(x), _gpu(y)
    parts = []
    prev = 0
    for r in range(ngpu):
        p = hc.Plan(D, "int64", ngpu, r)
        b, e = p.shard_info()
        assert b == prev and (b, e) == hc.shard_range(D, ngpu, r)
        prev = e
        zs = torch.empty(e - b, dtype=torch.int64, device="cuda")
        p.convolve_sharded(xs, ys, zs)
        parts.append(zs)
    assert prev == 3 ** D
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), full)


def test_host_entry_point(hc, orc):
    D = 13
    x, y = hcgen.make_pair(D, "float64", "exp_norm", 77)
    p = hc.Plan(D, "float64")
    zh = torch.empty(3 ** D, dtype=torch.float64).pin_memory()
    p.convolve_host(torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory(), zh)
    zd = _run(hc, x, y).cpu()
    assert torch.equal(zh, zd)
    _assert_close(zh.numpy(), orc.conv(x, y), x, y)
    # a shard of a 3-way split through the host entry point (chunked device output and
    # overlapped copies), int64 at D = 16 and D = 8 (single-level), = the device path
    for D, n, r in ((16, 3, 1), (8, 1, 0), (10, 3, 2), (12, 2, 1)):  # D = 12: the pair-split engine
        x, y = hcgen.make_pair(D, "int64", "uniform", 78 + D, -1000, 1000)
        p = hc.Plan(D, "int64", n, r)
        b, e = p.shard_info()
        zh = torch.empty(e - b, dtype=torch.int64).pin_memory()
        p.convolve_host(torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory(), zh)
        zd = torch.empty(e - b, dtype=torch.int64, device="cuda")
        p.convolve_sharded(_gpu(x), _gpu(y), zd)
        torch.cuda.synchronize()
        assert torch.equal(zh, zd.cpu())


@pytest.mark.parametrize("D", [3, 8, 11, 13, 16])
def test_delta_and_zero_inputs(hc, D):
    # degenerate inputs against their closed forms (no oracle): x = delta_a, y = delta_b gives
    # z = delta at T(a) + T(b) with T(i) = sum_b i_b 3^b (the carry-free sum, PAPER.md 359-365);
    # zero inputs give zero everywhere -- z is pre-filled with garbage so every cell must be written
    rng = np.random.default_rng(D)
    T = lambda i: sum(((int(i) >> b) & 1) * 3 ** b for b in range(D))
    for dtype, tdt in (("int64", torch.int64), ("float64", torch.float64)):
        for a, b in ((0, 0), ((1 << D) - 1, (1 << D) - 1), tuple(int(v) for v in rng.integers(0, 1 << D, 2))):
            x = np.zeros(1 << D, dtype=dtype)
            y = np.zeros(1 << D, dtype=dtype)
            x[a], y[b] = 3, -5
            z = torch.full((3 ** D,), 7, dtype=tdt, device="cuda")
            hc.Plan(D, dtype).convolve(_gpu(x), _gpu(y), z)
            torch.cuda.synchronize()
            want = np.zeros(3 ** D, dtype=dtype)
            want[T(a) + T(b)] = -15
            assert np.array_equal(z.cpu().numpy(), want), (dtype, a, b)
        zero = np.zeros(1 << D, dtype=dtype)
        z = torch.full((3 ** D,), 7, dtype=tdt, device="cuda")
        hc.Plan(D, dtype).convolve(_gpu(zero), _gpu(zero), z)
        torch.cuda.synchronize()
        assert not torch.any(z != 0)
    # batched (int64 D = 8: the 32-bit path), one delta cube and one zero cube
    if D == 8:
        xb = np.zeros((2, 256), dtype=np.int64)
        yb = np.zeros((2, 256), dtype=np.int64)
        xb[0, 200], yb[0, 77] = -4, 9
        zb = torch.full((2, 3 ** 8), 7, dtype=torch.int64, device="cuda")
        hc.convolve_batched(_gpu(xb), _gpu(yb), zb)
        torch.cuda.synchronize()
        want = np.zeros((2, 3 ** 8), dtype=np.int64)
        want[0, T(200) + T(77)] = -36
        assert np.array_equal(zb.cpu().numpy(), want)


def test_commutativity_int64(hc):
    D = 11
    x, y = hcgen.make_pair(D, "int64", "uniform", 9, -5000, 5000)
    assert torch.equal(_run(hc, x, y), _run(hc, y, x))


def test_errors(hc):
    with pytest.raises(hc.HCError):
        hc.Plan(0)
    with pytest.raises(hc.HCError):
        hc.Plan(hc.in_len(1) * 0 + 25)
    p = hc.Plan(4, "int64")
    x = torch.zeros(16, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        p.convolve(x, x, torch.empty(80, dtype=torch.int64, device="cuda"))
    # misaligned device pointer -> HC_ERR_ALIGN
    buf = torch.zeros(100, dtype=torch.int64, device="cuda")
    with pytest.raises(hc.HCError) as ei:
        p.convolve(buf[1:17], buf[1:17], torch.empty(81, dtype=torch.int64, device="cuda"))
    assert ei.value.code == 4
    # hc_conv1d: a multi-rank plan is rejected (HC_ERR_SHARD); the unfused route needs z_work
    import ctypes
    x13 = torch.zeros(1 << 13, dtype=torch.int64, device="cuda")
    out13 = torch.empty((2 << 13) - 1, dtype=torch.int64, device="cuda")
    with pytest.raises(hc.HCError) as ei:
        hc.conv1d(x13, x13, out13, plan=hc.Plan(13, "int64", 2, 0))
    assert ei.value.code == 9
    xf = torch.zeros(1 << 9, dtype=torch.float64, device="cuda")
    of = torch.empty((2 << 9) - 1, dtype=torch.float64, device="cuda")
    pf = hc.Plan(9, "float64")
    code = hc._lib.hc_conv1d(pf._h, ctypes.c_void_p(xf.data_ptr()), ctypes.c_void_p(xf.data_ptr()), None,
                             ctypes.c_void_p(of.data_ptr()), None, None)
    assert code == 3  # HC_ERR_NULL: fp64 needs the 3^D workspace


@pytest.mark.parametrize("D,dtype", [(13, "float64"), (14, "int64"), (15, "float64")])
def test_two_level_geometries(hc, orc, D, dtype):
    # D = 13: slab of 13 axes (M = 5), no top axes; 14: M = 6, k = 0; 15: M = 6, k = 1
    # (DESIGN.md §4): every cell against Algorithm 1
    if dtype == "int64":
        x, y = hcgen.make_pair(D, "int64", "uniform", 500 + D, -(1 << 20), 1 << 20)
    else:
        x, y = hcgen.make_pair(D, "float64", "exp_norm", 500 + D)
    got = _run(hc, x, y).cpu().numpy()
    _assert_close(got, orc.conv(x, y), x, y)


def test_d17_int64_sampled_and_ragged_shards(hc, orc):
    # k = 3 top axes, uneven shards (3 ranks over 27 slabs): concatenation = full output,
    # sampled cells (whole first/last slab tiles included) against the oracle
    D = 17
    x, y = hcgen.make_pair(D, "int64", "uniform", 1717, 0, 1 << 16)
    full = _run(hc, x, y)
    xs, ys = _gpu(x), _gpu(y)
    parts = []
    for r in range(3):
        p = hc.Plan(D, "int64", 3, r)
        b, e = p.shard_info()
        zs = torch.empty(e - b, dtype=torch.int64, device="cuda")
        p.convolve_sharded(xs, ys, zs)
        parts.append(zs)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), full)
    ks = _sample_cells(D, 20000, 17)
    got = full[torch.from_numpy(ks).cuda()].cpu().numpy()
    assert np.array_equal(got, orc.conv_cells(x, y, ks.astype(np.uint64)))


@pytest.mark.slow
def test_config_c5_d22_one_shard_of_eight(hc, orc):
    # BASELINE config 5 (D = 22 fp64, 251 GB of output) does not fit one GPU: compute the
    # shard of rank 5 of 8 (the launch configuration of the 8-GPU run) and check sampled
    # cells of it against the oracle, plus the shard's share of the mass.
    D, n, r = 22, 8, 5
    x, y = hcgen.config_inputs("c5_d22_f64")
    p = hc.Plan(D, "float64", n, r)
    b, e = p.shard_info()
    zs = torch.empty(e - b, dtype=torch.float64, device="cuda")
    p.convolve_sharded(_gpu(x), _gpu(y), zs)
    torch.cuda.synchronize()
    rng = np.random.default_rng(22)
    loc = np.unique(np.concatenate([rng.integers(0, e - b, 4000), np.arange(0, 3 ** 8),
                                    np.arange(e - b - 3 ** 8, e - b)]))
    got = zs[torch.from_numpy(loc).cuda()].cpu().numpy()
    want = orc.conv_cells(x, y, (loc + b).astype(np.uint64))
    _assert_close(got, want, x, y)
    assert torch.isfinite(zs).all()
    del zs


@pytest.mark.parametrize("D,k,dtype,nranks", [(11, 1, "int64", 2), (11, 2, "int64", 5), (12, 3, "int64", 3),
                                              (12, 4, "int64", 8), (10, 2, "float64", 4), (14, 4, "int64", 1),
                                              # D - k >= 13: the points run as one batch on the two-level engine
                                              (15, 2, "int64", 2), (15, 2, "int64", 3), (16, 2, "float64", 3), (17, 4, "int64", 8),
                                              # k = 5: 243 points, interpolated in shared memory
                                              (9, 5, "int64", 8), (13, 5, "float64", 3), (17, 5, "int64", 7)])
def test_evalpoint_variant_emulated_ranks(hc, orc, D, k, dtype, nranks):
    # north_star (4): every rank's local step, the exchange emulated on one device (each rank's
    # columns gathered from all ranks' w), the top-axes interpolation; the 3^k strided chunks
    # of each rank must equal Algorithm 1 (int64 bit-exact)
    if dtype == "int64":
        x, y = hcgen.make_pair(D, "int64", "uniform", 900 + D + k, -300, 300)
    else:
        x, y = hcgen.make_pair(D, "float64", "exp_norm", 900 + D + k)
    want = orc.conv(x, y)
    tdt = torch.int64 if dtype == "int64" else torch.float64
    xs, ys = _gpu(x), _gpu(y)
    nc, npnt = 3 ** (D - k), 3 ** k
    plans = [hc.EPPlan(D, k, dtype, nranks, r) for r in range(nranks)]
    W = torch.empty((npnt, nc), dtype=tdt, device="cuda")
    for p in plans:
        w = torch.empty((p.e1 - p.e0) * nc, dtype=tdt, device="cuda")
        p.local(xs, ys, w)
        W[p.e0:p.e1] = w.view(-1, nc)
    got = np.empty(3 ** D, dtype=want.dtype)
    for p in plans:
        wt = W[:, p.c0:p.c1].contiguous().view(-1)
        z = torch.empty_like(wt)
        p.finish(wt, z)
        torch.cuda.synchronize()
        got.reshape(npnt, nc)[:, p.c0:p.c1] = z.view(npnt, -1).cpu().numpy()
    _assert_close(got, want, x, y)
    # f3: the exchange fused into the interpolation -- every rank reads the owners' buffers
    ws = [W[p.e0:p.e1].contiguous().view(-1) for p in plans]
    got2 = np.empty(3 ** D, dtype=want.dtype)
    for p in plans:
        z = torch.empty(npnt * (p.c1 - p.c0), dtype=tdt, device="cuda")
        p.finish_peer(ws, z)
        torch.cuda.synchronize()
        got2.reshape(npnt, nc)[:, p.c0:p.c1] = z.view(npnt, -1).cpu().numpy()
    assert np.array_equal(got2, got)
    if nranks == 1:  # world 1: ep_exchange is the identity copy
        p = plans[0]
        w = torch.empty(npnt * nc, dtype=tdt, device="cuda")
        p.local(xs, ys, w)
        wt = torch.empty_like(w)
        hc.ep_exchange(w, wt, D, k, 0, 1)
        z = torch.empty_like(w)
        p.finish(wt, z)
        torch.cuda.synchronize()
        _assert_close(z.cpu().numpy(), want, x, y)


@pytest.mark.parametrize("D,k,nranks", [(17, 2, 2), (18, 3, 4), (19, 5, 8)])
def test_evalpoint_batched_slab_points_sampled(hc, orc, D, k, nranks):
    # D - k = 15: each point is a two-level convolution with k' = 1 direct top axis (3 slabs), and
    # all of a rank's points run as one batch of points x slabs through the slab engine; the
    # evaluation-domain result of point e is checked against the (D-k)-dimensional oracle
    # convolution of the point's evaluated inputs (forward over the top axes, PAPER.md 186-189),
    # and the finished output on sampled cells against Algorithm 1
    x, y = hcgen.make_pair(D, "int64", "uniform", 5100 + D, -500, 500)
    L, nc, npnt = D - k, 3 ** (D - k), 3 ** k
    xs, ys = _gpu(x), _gpu(y)
    plans = [hc.EPPlan(D, k, "int64", nranks, r) for r in range(nranks)]
    W = torch.empty((npnt, nc), dtype=torch.int64, device="cuda")
    for p in plans:
        w = torch.empty((p.e1 - p.e0) * nc, dtype=torch.int64, device="cuda")
        p.local(xs, ys, w)
        W[p.e0:p.e1] = w.view(-1, nc)
    torch.cuda.synchronize()
    xr, yr = x.reshape(2 ** k, 2 ** L), y.reshape(2 ** k, 2 ** L)
    for e in (0, 1, npnt // 2 + 1, npnt - 1):   # points owned by different ranks
        t, base, free = e, 0, 0
        for a in range(k):
            base |= (1 << a) if t % 3 == 2 else 0
            free |= (1 << a) if t % 3 == 1 else 0
            t //= 3
        subs = [s for s in range(2 ** k) if s & ~free == 0]
        xe = sum(xr[base | s] for s in subs)
        ye = sum(yr[base | s] for s in subs)
        ks = np.random.default_rng(e).integers(0, nc, 4000).astype(np.uint64)
        assert np.array_equal(W[e].cpu().numpy()[ks.astype(np.int64)], orc.conv_cells(xe, ye, ks)), e
    ks = np.random.default_rng(D).integers(0, 3 ** D, 20000)
    got = np.empty(ks.size, dtype=np.int64)
    for p in plans:
        wt = W[:, p.c0:p.c1].contiguous().view(-1)
        z = torch.empty_like(wt)
        p.finish(wt, z)
        torch.cuda.synchronize()
        zz = z.view(npnt, -1).cpu().numpy()
        col, row = ks % nc, ks // nc
        m = (col >= p.c0) & (col < p.c1)
        got[m] = zz[row[m], col[m] - p.c0]
    assert np.array_equal(got, orc.conv_cells(x, y, ks.astype(np.uint64)))


def test_output_at_odd_element_offset(hc, orc):
    # z only needs element (8-byte) alignment: write into a view that starts one element in
    for D in (7, 9, 13):
        x, y = hcgen.make_pair(D, "int64", "uniform", 4242 + D, -50, 50)
        buf = torch.zeros(3 ** D + 1, dtype=torch.int64, device="cuda")
        hc.Plan(D, "int64").convolve(_gpu(x), _gpu(y), buf[1:])
        torch.cuda.synchronize()
        assert int(buf[0]) == 0
        assert np.array_equal(buf[1:].cpu().numpy(), orc.conv(x, y))


# ---- applications ---------------------------------------------------------
@pytest.fixture(scope="module")
def apps(orc):
    import oracle.apps as a
    return a


@pytest.mark.parametrize("D,dtype", [(1, "int64"), (3, "int64"), (7, "float64"), (9, "int64"), (12, "float64"),
                                     (13, "int64")])
def test_difference_pmf(hc, apps, D, dtype):
    # f4: P(X - Y = k - 1) against its definition (every pair, digit-wise difference)
    if dtype == "int64":
        x, y = hcgen.make_pair(D, "int64", "uniform", 9100 + D, -100, 100)
    else:
        x, y = hcgen.make_pair(D, "float64", "exp_norm", 9100 + D)
    tdt = torch.int64 if dtype == "int64" else torch.float64
    z = torch.empty(3 ** D, dtype=tdt, device="cuda")
    hc.Plan(D, dtype).convolve_difference(_gpu(x), _gpu(y), z)
    torch.cuda.synchronize()
    _assert_close(z.cpu().numpy(), apps.difference_pmf(x, y), x, y)


@pytest.mark.parametrize("D", [1, 4, 8, 9, 11, 13, 14, 15])
def test_conv1d_via_carries_int64(hc, D):
    # f1: carry-free convolution + carries = the ordinary 1-D convolution (numpy's definition)
    x = hcgen.uniform_int(9200 + D, 0, 1 << D, -10 ** 6, 10 ** 6)
    y = hcgen.uniform_int(9200 + D, 1, 1 << D, -10 ** 6, 10 ** 6)
    out = hc.conv1d(_gpu(x), _gpu(y))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), np.convolve(x, y))


def test_carries_fp64_and_d20_sampled(hc, apps, orc):
    # fp64: the carries of the GPU hypercube output equal the oracle's carries of the oracle's
    # convolution; D = 20 int64: sampled m against sum_i x[i] y[m - i]
    D = 10
    x, y = hcgen.make_pair(D, "float64", "exp_norm", 9300)
    out = hc.conv1d(_gpu(x), _gpu(y)).cpu().numpy()
    want = apps.conv1d_carryfree_then_carries(x, y)
    assert np.max(np.abs(out - want)) <= 1e-12 * float(x.sum() * y.sum())
    D = 20
    x = hcgen.uniform_int(9301, 0, 1 << D, 0, 1 << 16)
    y = hcgen.uniform_int(9301, 1, 1 << D, 0, 1 << 16)
    out = hc.conv1d(_gpu(x), _gpu(y)).cpu().numpy()
    rng = np.random.default_rng(20)
    for m in list(rng.integers(0, (2 << D) - 1, 200)) + [0, 1, (1 << D) - 1, (2 << D) - 2]:
        lo, hi = max(0, m - (1 << D) + 1), min(m, (1 << D) - 1)
        i = np.arange(lo, hi + 1)
        assert out[m] == int((x[i].astype(object) * y[m - i].astype(object)).sum())


def _power_domain(E, mx, my, p):
    return np.where(E > 0, (E / (mx * my)) ** p, 0.0)


@pytest.mark.parametrize("D,p", [(6, 2.0), (8, 16.0), (10, 64.0), (13, 8.0)])
def test_maxconv_pnorm_estimate(hc, apps, D, p):
    # f2: the GPU p-norm estimate against the oracle's (same formula on Algorithm 1).  The sum
    # of p-th powers goes through the hot path, whose tolerance is absolute (1e-12 x the scaled
    # masses, R4): compare there on every cell, and compare the estimates relatively
    # on the cells whose power sum stands above that noise (R11).
    x = hcgen.uniform_int(9400 + D, 0, 1 << D, 0, 1000).astype(np.float64)
    y = hcgen.uniform_int(9400 + D, 1, 1 << D, 0, 1000).astype(np.float64)
    z = torch.empty(3 ** D, dtype=torch.float64, device="cuda")
    hc.Plan(D, "float64").maxconv_pnorm(_gpu(x), _gpu(y), z, p)
    torch.cuda.synchronize()
    got, want = z.cpu().numpy(), apps.maxconv_pnorm(x, y, p)
    mx, my = x.max(), y.max()
    mass = float(((x / mx) ** p).sum() * ((y / my) ** p).sum())
    sg, sw = _power_domain(got, mx, my, p), _power_domain(want, mx, my, p)
    assert np.max(np.abs(sg - sw)) <= 1e-12 * mass
    good = sw >= 1e-6 * mass
    assert good.sum() > 0
    assert np.allclose(got[good], want[good], rtol=1e-10, atol=0)
    M = apps.maxconv_exact(x, y)
    assert (got[good] >= M[good] * (1 - 1e-10)).all() and (got[good] <= M[good] * 2.0 ** (D / p) * (1 + 1e-10)).all()


def test_maxconv_pnorm_exact_rounding(hc, apps):
    # PAPER.md 346-352: bounded integers and p with M (n^(1/p) - 1) < 0.5 -> rounding gives the
    # exact max-convolution, on every cell whose power sum the fp64 pipeline resolves
    # (R11), which includes the global maximum
    D = 8
    x = hcgen.uniform_int(9500, 0, 1 << D, 0, 3).astype(np.float64)
    y = hcgen.uniform_int(9500, 1, 1 << D, 0, 3).astype(np.float64)
    p = float(np.ceil(np.log(2.0 ** D) / np.log(1 + 0.5 / 9.0))) + 1
    z = torch.empty(3 ** D, dtype=torch.float64, device="cuda")
    hc.Plan(D, "float64").maxconv_pnorm(_gpu(x), _gpu(y), z, p, round_to_int=True)
    torch.cuda.synchronize()
    got, M = z.cpu().numpy(), apps.maxconv_exact(x, y)
    mx, my = x.max(), y.max()
    mass = float(((x / mx) ** p).sum() * ((y / my) ** p).sum())
    resolved = (M / (mx * my)) ** p >= 1e-6 * mass
    assert resolved[np.argmax(M)] and resolved.sum() > 0
    assert np.array_equal(got[resolved], M[resolved])


def test_scheduler_race_stress(hc, orc):
    # the persistent kernels hand work out through atomics, mbarriers and completion
    # counters: repeated runs (whole outputs and uneven shards) must all be bit-identical to
    # Algorithm 1 -- a race in the schedule would show up as run-to-run differences
    for D, seed in ((13, 1), (15, 2), (16, 3)):
        x, y = hcgen.make_pair(D, "int64", "uniform", 6000 + seed, -(1 << 20), 1 << 20)
        want = orc.conv(x, y)
        xs, ys = _gpu(x), _gpu(y)
        p = hc.Plan(D, "int64")
        z = torch.empty(3 ** D, dtype=torch.int64, device="cuda")
        for _ in range(6):
            z.fill_(-1)
            p.convolve(xs, ys, z)
            torch.cuda.synchronize()
            assert np.array_equal(z.cpu().numpy(), want)
        for n in {13: (), 15: (2, 3), 16: (2, 5)}[D]:  # shards need 3^k >= n slabs
            parts = []
            for r in range(n):
                pr = hc.Plan(D, "int64", n, r)
                b, e = pr.shard_info()
                zs = torch.empty(e - b, dtype=torch.int64, device="cuda")
                pr.convolve_sharded(xs, ys, zs)
                parts.append(zs)
            torch.cuda.synchronize()
            assert np.array_equal(torch.cat(parts).cpu().numpy(), want)


def test_slab_ring_lag_clamped():
    # HC_SLAB_LAG beyond the fused-carry slab ring (4 buffers) is clamped to 3: the 1-D
    # convolution through the ring still equals numpy's (no deadlock, no overwritten slot)
    import subprocess
    import sys
    import os
    code = (
        "import sys; sys.path.insert(0, '.'); import numpy as np, torch, hcgen;"
        "import paper_1608_00206_b200.hc as hc\n"
        "for D in (13, 16):\n"
        "    x, y = hcgen.make_pair(D, 'int64', 'uniform', 7300 + D, -999, 999)\n"
        "    out = hc.conv1d(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())\n"
        "    torch.cuda.synchronize(); assert np.array_equal(out.cpu().numpy(), np.convolve(x, y)), D\n"
        "print('ok')\n")
    env = dict(os.environ, HC_SLAB_LAG="4")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("env", [{"HC_SLAB_LAG": "2"}, {"HC_ENGINE": "slabx"}, {"HC_ENGINE": "slabx", "HC_SLABX_LAG": "1"},
                                 {"HC_P2_HEAD": "243"}, {"HC_KEEP_POLICY": "1", "HC_P2_PREFETCH": "1"},
                                 {"HC_NARROW": "0"}, {"HC_PAIR_SPLIT": "0"}])
def test_engine_variants_by_env(env):
    # engine knobs are environment variables read once per process: run them in a child
    # process against the oracle
    import subprocess
    import sys
    import os
    code = (
        "import sys; sys.path.insert(0, '.'); import numpy as np, torch, hcgen, oracle;"
        "import paper_1608_00206_b200.hc as hc; oracle.build()\n"
        "for D in (9, 11, 13, 15, 16):\n"
        "    x, y = hcgen.make_pair(D, 'int64', 'uniform', 7100 + D, -999, 999)\n"
        "    z = torch.empty(3 ** D, dtype=torch.int64, device='cuda')\n"
        "    hc.Plan(D, 'int64').convolve(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), z)\n"
        "    torch.cuda.synchronize(); assert np.array_equal(z.cpu().numpy(), oracle.conv(x, y)), D\n"
        "xb, yb = hcgen.make_batched_fast(5, 8, 0, 255, 71)\n"
        "zb = torch.empty((5, 6561), dtype=torch.int64, device='cuda')\n"
        "hc.convolve_batched(torch.from_numpy(xb).cuda(), torch.from_numpy(yb).cuda(), zb)\n"
        "torch.cuda.synchronize(); assert np.array_equal(zb.cpu().numpy(), oracle.conv_batched(xb, yb))\n"
        "D = 17\n"  # k = 3 top axes: 27 slabs, 3-way shards concatenate to the full output
        "x, y = hcgen.make_pair(D, 'float64', 'exp_norm', 7117)\n"
        "xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()\n"
        "z = torch.empty(3 ** D, dtype=torch.float64, device='cuda'); hc.Plan(D, 'float64').convolve(xg, yg, z)\n"
        "parts = []\n"
        "for r in range(3):\n"
        "    p = hc.Plan(D, 'float64', 3, r); b, e = p.shard_info()\n"
        "    zs = torch.empty(e - b, dtype=torch.float64, device='cuda'); p.convolve_sharded(xg, yg, zs); parts.append(zs)\n"
        "torch.cuda.synchronize(); assert torch.equal(torch.cat(parts), z)\n"
        "ks = np.random.default_rng(17).integers(0, 3 ** D, 20000)\n"
        "err = np.max(np.abs(z[torch.from_numpy(ks).cuda()].cpu().numpy() - oracle.conv_cells(x, y, ks.astype(np.uint64))))\n"
        "assert err <= 1e-12, err\n"
        "print('ok')\n")
    env = dict(os.environ, **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("D", [3, 9, 11, 13, 15])
def test_int64_full_range_wraparound(hc, orc, D):
    # inputs over the whole 64-bit range: every product and every interpolation wraps; the
    # pipeline is a ring homomorphism mod 2^64 (R3), so it must agree bit for bit
    # with Algorithm 1 computed mod 2^64 -- through the single-level, two-level and batched
    # engines, a shard, and the differences entry point
    x = hcgen.splitmix64(8800 + D, 0, 1 << D).view(np.int64)
    y = hcgen.splitmix64(8800 + D, 1, 1 << D).view(np.int64)
    want = orc.conv(x, y)
    got = _run(hc, x, y).cpu().numpy()
    assert np.array_equal(got, want)
    xb = np.stack([x, y])
    yb = np.stack([y, x])
    zb = torch.empty((2, 3 ** D), dtype=torch.int64, device="cuda")
    hc.convolve_batched(_gpu(xb), _gpu(yb), zb)
    torch.cuda.synchronize()
    assert np.array_equal(zb.cpu().numpy(), orc.conv_batched(xb, yb))
    if D >= 15:
        p = hc.Plan(D, "int64", 2, 1)
        b, e = p.shard_info()
        zs = torch.empty(e - b, dtype=torch.int64, device="cuda")
        p.convolve_sharded(_gpu(x), _gpu(y), zs)
        torch.cuda.synchronize()
        assert np.array_equal(zs.cpu().numpy(), want[b:e])
    zd = torch.empty(3 ** D, dtype=torch.int64, device="cuda")
    hc.Plan(D, "int64").convolve_difference(_gpu(x), _gpu(y), zd)
    torch.cuda.synchronize()
    mask = (1 << D) - 1
    yf = y[np.bitwise_xor(np.arange(1 << D), mask)]
    assert np.array_equal(zd.cpu().numpy(), orc.conv(x, yf))


def test_max_dimension_d24_shard(hc, orc):
    # HC_MAX_D = 24 (3^24 = 2.8e11 entries, 2.3 TB of output): one shard of a 128-way output
    # split, int64 (bit-exact), sampled cells plus the shard's first and last tiles
    D, n, r = 24, 128, 77
    x = hcgen.uniform_int(2424, 0, 1 << D, 0, 255)
    y = hcgen.uniform_int(2424, 1, 1 << D, 0, 255)
    p = hc.Plan(D, "int64", n, r)
    b, e = p.shard_info()
    assert 0 < e - b < 3 ** D // 64
    zs = torch.empty(e - b, dtype=torch.int64, device="cuda")
    p.convolve_sharded(_gpu(x), _gpu(y), zs)
    torch.cuda.synchronize()
    rng = np.random.default_rng(24)
    loc = np.unique(np.concatenate([rng.integers(0, e - b, 3000), np.arange(0, 3 ** 8),
                                    np.arange(e - b - 3 ** 8, e - b)]))
    got = zs[torch.from_numpy(loc).cuda()].cpu().numpy()
    want = orc.conv_cells(x, y, (loc + b).astype(np.uint64))
    assert np.array_equal(got, want)
    p.close()
    del zs


def test_c_example_program(tmp_path):
    # examples/hc_example.c: a plain C program using the ABI (host-buffer entry point) and
    # checking D = 10 against the definition by brute force
    import subprocess
    from test_lib_cpu import _build_example
    exe = _build_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 of 59049 output entries differ" in r.stdout


@pytest.mark.parametrize("D", [13, 16])
def test_conv1d_fused_equals_convolve_then_carries(hc, D):
    # int64, D >= 13: hc_conv1d fuses the carries into pass 2 (atomics into the bins); it must
    # equal the unfused route (hc_convolve, then hc_apply_carries) bit for bit, including
    # values that wrap
    x = hcgen.splitmix64(7700 + D, 0, 1 << D).view(np.int64)
    y = hcgen.splitmix64(7700 + D, 1, 1 << D).view(np.int64)
    xg, yg = _gpu(x), _gpu(y)
    fused_ring = hc.conv1d(xg, yg)  # pass-1 tiles in the plan's ring of slab buffers
    z = torch.empty(3 ** D, dtype=torch.int64, device="cuda")
    fused_inplace = hc.conv1d(xg, yg, z_work=z)  # tiles in place in z
    hc.Plan(D, "int64").convolve(xg, yg, z)
    ref = torch.empty((2 << D) - 1, dtype=torch.int64, device="cuda")
    hc.apply_carries(D, z, ref)
    torch.cuda.synchronize()
    assert torch.equal(fused_ring, ref)
    assert torch.equal(fused_inplace, ref)


def test_conv1d_d21_without_z(hc):
    # int64 D = 21: the carry-free output would be 3^21 x 8 B = 84 GB; the fused path keeps only
    # a ring of four slabs and the 2^22 - 1 carry bins.  Sampled m against sum_i x[i] y[m - i].
    D = 21
    x = hcgen.uniform_int(2121, 0, 1 << D, 0, (1 << 16) - 1)
    y = hcgen.uniform_int(2121, 1, 1 << D, 0, (1 << 16) - 1)
    free0 = torch.cuda.mem_get_info()[0]
    out = hc.conv1d(_gpu(x), _gpu(y)).cpu().numpy()
    assert torch.cuda.mem_get_info()[0] > free0 - (2 << 30)  # far less than z would take
    rng = np.random.default_rng(21)
    for m in list(rng.integers(0, (2 << D) - 1, 150)) + [0, 1, (1 << D) - 1, (2 << D) - 2]:
        lo, hi = max(0, m - (1 << D) + 1), min(m, (1 << D) - 1)
        i = np.arange(lo, hi + 1)
        assert out[m] == int((x[i].astype(object) * y[m - i].astype(object)).sum())


def test_property_random_shapes(hc, orc):
    # property check over random small problems: D, dtype, value range, batch size and shard
    # split drawn from a seeded generator; every output against Algorithm 1
    rng = np.random.default_rng(4242)
    for trial in range(24):
        D = int(rng.integers(1, 13))
        dtype = "int64" if rng.random() < 0.6 else "float64"
        if dtype == "int64":
            lo = -int(rng.integers(0, 1 << 30))
            x, y = hcgen.make_pair(D, "int64", "uniform", 9000 + trial, lo, int(rng.integers(1, 1 << 30)))
        else:
            x, y = hcgen.make_pair(D, "float64", "exp_norm", 9000 + trial)
        want = orc.conv(x, y)
        _assert_close(_run(hc, x, y).cpu().numpy(), want, x, y)
        B = int(rng.integers(1, 5))
        xb = np.stack([np.roll(x, b) for b in range(B)])
        yb = np.stack([np.roll(y, 3 * b) for b in range(B)])
        zb = torch.empty((B, 3 ** D), dtype=_gpu(x).dtype, device="cuda")
        hc.convolve_batched(_gpu(xb), _gpu(yb), zb)
        torch.cuda.synchronize()
        _assert_close(zb.cpu().numpy(), orc.conv_batched(xb, yb), xb, yb)
