"""Dev check of the two-level engines: parity at small D against the oracle, then D=20 timing."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import hcgen, oracle
import paper_1608_00206_b200.hc as hc

def run(D, x, y):
    z = torch.empty(3 ** D, dtype=torch.float64 if x.dtype == np.float64 else torch.int64, device='cuda')
    hc.Plan(D, str(x.dtype)).convolve(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), z)
    torch.cuda.synchronize()
    return z

ok = True
for D, dt in ((13, 'int64'), (14, 'float64'), (15, 'int64'), (16, 'float64'), (17, 'int64')):
    if dt == 'int64':
        x, y = hcgen.make_pair(D, dt, 'uniform', 900 + D, -(1 << 20), 1 << 20)
    else:
        x, y = hcgen.make_pair(D, dt, 'exp_norm', 900 + D)
    t0 = time.time()
    z = run(D, x, y).cpu().numpy()
    want = oracle.conv(x, y)
    if dt == 'int64':
        bad = int(np.count_nonzero(z != want))
        print(f"D={D} {dt}: {bad} cells differ ({time.time()-t0:.1f}s)", flush=True)
        ok &= bad == 0
    else:
        err = float(np.max(np.abs(z - want)))
        print(f"D={D} {dt}: max err {err:.3e} ({time.time()-t0:.1f}s)", flush=True)
        ok &= err <= 1e-12
print("parity", "OK" if ok else "FAIL", flush=True)
if not ok:
    sys.exit(1)
# D = 20 timing
x, y = hcgen.config_inputs('c4_d20_f64')
xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
p = hc.Plan(20, 'float64')
z = torch.empty(3 ** 20, dtype=torch.float64, device='cuda')
for _ in range(2):
    p.convolve(xg, yg, z)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p.convolve(xg, yg, z); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("D=20 fp64 ms:", " ".join(f"{t:.2f}" for t in ts), f"min {min(ts):.3f}", flush=True)
ks = np.random.default_rng(5).integers(0, 3 ** 20, 20000)
got = z[torch.from_numpy(ks).cuda()].cpu().numpy()
want = oracle.conv_cells(x, y, ks.astype(np.uint64))
print("D=20 sampled max err", float(np.max(np.abs(got - want))), flush=True)
