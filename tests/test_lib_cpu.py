"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/hc.h declares, validates arguments, and its host-only sharding logic partitions
the output correctly.  No compute call is made here (no GPU)."""
import os
import subprocess

import pytest

import hcgen  # noqa: F401  (keeps the import graph honest: tests may use generators)


@pytest.fixture(scope="module")
def hc():
    import paper_1608_00206_b200.build as b
    b.build()
    import paper_1608_00206_b200.hc as hcmod
    return hcmod


def test_exports_every_declared_symbol(hc):
    names = hc.exported_symbols()
    assert len(names) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", hc.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_lengths(hc):
    assert hc.in_len(1) == 2 and hc.out_len(1) == 3
    assert hc.in_len(20) == 1 << 20 and hc.out_len(20) == 3 ** 20
    assert hc.out_len(22) == 3 ** 22 and hc.out_len(0) == 0 and hc.out_len(25) == 0


def test_status_strings(hc):
    for code in (0, 1, 2, 3, 4, 5, 6, 7, 9):
        assert hc._lib.hc_status_str(code)


def test_plan_argument_errors_before_device(hc):
    # D and dtype are validated before the device check
    for D, dt, code in ((0, 1, 1), (25, 1, 1), (5, 7, 2)):
        h = hc._P()
        assert hc._lib.hc_plan_create(hc.ctypes.byref(h), D, dt, 1, 0) == code
    h = hc._P()
    assert hc._lib.hc_plan_create(hc.ctypes.byref(h), 5, 1, 2, 2) == 9   # rank >= ngpu
    assert hc._lib.hc_plan_create(None, 5, 1, 1, 0) == 3


def test_plan_without_device_fails_loudly(hc):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(hc.HCError) as ei:
        hc.Plan(10)
    assert ei.value.code == 5


ALPHA = 11.0  # compute_cuts' fixed cost per slab, in pairs (fitted: profiles/r02_shard_balance.txt)


def _slab_cost(t, k):
    ones = 0
    for _ in range(k):
        ones += t % 3 == 1
        t //= 3
    return ALPHA + 2 ** ones


def _unit_axes(D):
    # DESIGN.md §4 geometry: single level (tile of min(D, 8) axes) for D <= 12, otherwise a
    # two-level slab of min(D, 14) axes; the remaining top axes use the direct split
    return min(D, 8) if D <= 12 else min(D, 14)


@pytest.mark.parametrize("D", [9, 12, 16, 20, 22])
@pytest.mark.parametrize("ngpu", [1, 2, 3, 4, 8])
def test_shard_ranges_partition(hc, D, ngpu):
    s = _unit_axes(D)
    if ngpu > 3 ** (D - s):
        with pytest.raises(hc.HCError):
            hc.shard_range(D, ngpu, 0)
        return
    ranges = [hc.shard_range(D, ngpu, r) for r in range(ngpu)]
    assert ranges[0][0] == 0 and ranges[-1][1] == 3 ** D
    for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
        assert e0 == b1
    tile = 3 ** s
    for b, e in ranges:
        assert b % tile == 0 and e % tile == 0 and e > b
    if D <= 16 and ngpu > 1:
        # balance: per-rank cost within one heaviest slab of the ideal share
        k = D - s
        costs = [sum(_slab_cost(t, k) for t in range(b // tile, e // tile)) for b, e in ranges]
        ideal = sum(costs) / ngpu
        assert max(costs) - ideal <= ALPHA + 2 ** k


def test_shard_errors(hc):
    with pytest.raises(hc.HCError):
        hc.shard_range(20, 0, 0)
    with pytest.raises(hc.HCError):
        hc.shard_range(20, 2, 2)
    with pytest.raises(hc.HCError):
        hc.shard_range(8, 2, 0)   # a single slab cannot be split


@pytest.mark.parametrize("D,k", [(6, 1), (12, 3), (20, 4), (22, 4), (20, 5)])
def test_ep_ranges_partition(hc, D, k):
    # evaluation-point variant (hc_ep_range): points and columns are split contiguously,
    # disjointly, in rank order, sizes within one of each other
    for n in [1, 2, 3, 8, 3 ** k]:
        if n > 3 ** k:
            continue
        rs = [hc.ep_range(D, k, n, r) for r in range(n)]
        for which, total in ((0, 3 ** k), (1, 3 ** (D - k))):
            segs = [r[which] for r in rs]
            assert segs[0][0] == 0 and segs[-1][1] == total
            assert all(segs[i][1] == segs[i + 1][0] for i in range(n - 1))
            sizes = [b - a for a, b in segs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(hc.HCError):
        hc.ep_range(D, k, 3 ** k + 1, 0)
    with pytest.raises(hc.HCError):
        hc.ep_range(D, 6, 1, 0)   # k <= 5 (EP_MAX_K)


def _build_example(tmp_path):
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1608_00206_b200")
    exe = str(tmp_path / "hc_example")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Wextra", "-Werror", "-std=c99", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "hc_example.c"), "-L", libdir, "-lhc",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    return exe


def test_c_example_builds_against_the_header(tmp_path):
    # the boundary is plain C: the example compiles with gcc -std=c99 -Werror and links
    # against libhc.so; without a GPU it must fail loudly (no CPU fallback)
    import subprocess
    exe = _build_example(tmp_path)
    import torch
    if not torch.cuda.is_available():
        r = subprocess.run([exe], capture_output=True, text=True)
        assert r.returncode == 1 and "no usable CUDA device" in r.stderr
