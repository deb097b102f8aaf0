"""single-level int64 D = 9..12: (tile, pair) items with atomics vs one item per tile (HC_PAIR_SPLIT)"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import hcgen
import paper_1608_00206_b200.hc as hc
flush = torch.empty(4 * 126 * 2 ** 20, dtype=torch.uint8, device="cuda")
for D in (9, 10, 11, 12):
    x, y = hcgen.make_pair(D, "int64", "uniform", 40 + D, 0, 9)
    xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    p = hc.Plan(D, "int64")
    z = torch.empty(3 ** D, dtype=torch.int64, device="cuda")
    for _ in range(3): p.convolve(xg, yg, z)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.convolve(xg, yg, z); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"D={D} int64 L2-flushed: min {min(ts)*1e3:.1f} us med {np.median(ts)*1e3:.1f} us", flush=True)
