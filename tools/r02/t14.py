"""per-output cost of the int64 / fp64 two-level engine vs direct-split pairs (D = 14..19)"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import hcgen
import paper_1608_00206_b200.hc as hc
for dt in ("int64", "float64"):
    for D in range(14, 20):
        if dt == "int64":
            x, y = hcgen.make_pair(D, "int64", "uniform", 77 + D, 0, (1 << 16) - 1)
        else:
            x, y = hcgen.make_pair(D, "float64", "exp_norm", 77 + D)
        xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        p = hc.Plan(D, dt)
        z = torch.empty(3 ** D, dtype=xg.dtype, device="cuda")
        for _ in range(3): p.convolve(xg, yg, z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record(); p.convolve(xg, yg, z); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        t = min(ts)
        k = max(D - 14, 0)
        print(f"{dt} D={D} k={k} pairs/out={(4/3)**k:.2f} ms={t:.3f} ns/out={t*1e6/3**D:.4f} clk/out/SM={t*1e-3*148*1.965e9/3**D:.3f}", flush=True)
