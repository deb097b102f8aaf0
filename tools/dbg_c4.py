import sys, numpy as np, torch
sys.path.insert(0, '.')
import hcgen, oracle
import paper_1608_00206_b200.hc as hc
D = int(sys.argv[1]) if len(sys.argv) > 1 else 20
x, y = hcgen.make_pair(D, "float64", "exp_norm", 1004)
p = hc.Plan(D, "float64")
xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
z = torch.empty(3 ** D, dtype=torch.float64, device="cuda"); p.convolve(xg, yg, z)
z2 = torch.empty_like(z); p.convolve(xg, yg, z2); torch.cuda.synchronize()
print("bit-identical rerun:", torch.equal(z, z2), "ndiff", int((z != z2).sum()))
rng = np.random.default_rng(0)
ks = rng.integers(0, 3 ** D, size=20000).astype(np.uint64)
got = z[torch.from_numpy(ks.astype(np.int64)).cuda()].cpu().numpy()
want = oracle.conv_cells(x, y, ks)
err = np.abs(got - want)
print("max err", err.max(), "n bad", int((err > 1e-12).sum()))
bad = np.nonzero(err > 1e-12)[0][:10]
for b in bad:
    k = int(ks[b]); print(k, k // 3 ** 14, (k // 6561) % 729, k % 6561, got[b], want[b])
print("mass", float(z.sum()), float(x.sum() * y.sum()))
