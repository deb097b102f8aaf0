"""Development aid: repeated D = 20 runs must be bit-identical (fp64 plain path, int64 fused
conv1d in ring mode), and sharded D = 18 runs concatenate to the whole output."""
import sys
import torch
sys.path.insert(0, '.')
import hcgen
import paper_1608_00206_b200.hc as hc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x, y = hcgen.config_inputs("c4_d20_f64")
xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
p = hc.Plan(20, "float64")
z = torch.empty(3 ** 20, dtype=torch.float64, device="cuda")
p.convolve(xg, yg, z)
ref = z.view(torch.int64)[::997].clone()
refsum = float(z.sum())
for i in range(n):
    z.fill_(float("nan"))
    p.convolve(xg, yg, z)
    assert torch.equal(z.view(torch.int64)[::997], ref) and float(z.sum()) == refsum, f"fp64 run {i} differs"
print(f"fp64 D=20: {n + 1} runs bit-identical (sampled), sum {refsum:.17g}")
xi = torch.from_numpy(hcgen.uniform_int(5, 0, 1 << 20, 0, (1 << 16) - 1)).cuda()
yi = torch.from_numpy(hcgen.uniform_int(5, 1, 1 << 20, 0, (1 << 16) - 1)).cuda()
pi = hc.Plan(20, "int64")
o1 = hc.conv1d(xi, yi, plan=pi)
for i in range(n):
    assert torch.equal(hc.conv1d(xi, yi, plan=pi), o1), f"conv1d run {i} differs"
assert (int(o1.sum()) - int(xi.sum()) * int(yi.sum())) % (1 << 64) == 0  # mass, mod 2^64
print(f"conv1d D=20 ring: {n + 1} runs identical, mass ok")
D = 18
x8, y8 = hcgen.make_pair(D, "int64", "uniform", 18, -1000, 1000)
x8g, y8g = torch.from_numpy(x8).cuda(), torch.from_numpy(y8).cuda()
full = torch.empty(3 ** D, dtype=torch.int64, device="cuda")
hc.Plan(D, "int64").convolve(x8g, y8g, full)
for nr in (2, 5, 7):
    parts = []
    for r in range(nr):
        q = hc.Plan(D, "int64", nr, r)
        b, e = q.shard_info()
        zs = torch.empty(e - b, dtype=torch.int64, device="cuda")
        q.convolve_sharded(x8g, y8g, zs)
        parts.append(zs)
    assert torch.equal(torch.cat(parts), full), f"{nr} shards differ"
print("D=18 int64: 2/5/7-way shards concatenate to the whole output")
