import sys, numpy as np, torch
sys.path.insert(0, '.')
import hcgen, oracle
import paper_1608_00206_b200.hc as hc
fl = torch.empty(4 * 126 * 2**20, dtype=torch.uint8, device='cuda')
for D in (9, 10, 11, 12):
    x, y = hcgen.make_pair(D, 'int64', 'uniform', 1001, 0, 9)
    xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    p = hc.Plan(D, 'int64')
    z = torch.empty(3 ** D, dtype=torch.int64, device='cuda')
    p.convolve(xg, yg, z); torch.cuda.synchronize()
    ok = np.array_equal(z.cpu().numpy(), oracle.conv(x, y))
    ts = []
    for _ in range(20):
        fl.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.convolve(xg, yg, z); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    print(f"D={D} parity {ok} us median {np.median(ts):.1f} min {min(ts):.1f}", flush=True)
