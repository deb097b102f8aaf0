"""Quick device timing of the hot configs (development aid; bench.py is the contract)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import hcgen
import paper_1608_00206_b200.hc as hc

def t_ms(fn, reps=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts), float(np.median(ts))

which = sys.argv[1:] or ["c2", "c3", "c1", "c4"]
if "c2" in which:
    x, y = hcgen.config_inputs("c2_b65536_d8_i64")
    xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    z = torch.empty((65536, 6561), dtype=torch.int64, device="cuda")
    mn, md = t_ms(lambda: hc.convolve_batched(xg, yg, z))
    print(f"c2 batched D=8 int64: min {mn:.3f} ms med {md:.3f} ms  ({z.numel()*8/mn/1e6:.0f} GB/s out)")
for name, cfg, D in (("c1", "c1_d10_i64", 10), ("c3", "c3_d16_i64", 16), ("c4", "c4_d20_f64", 20)):
    if name not in which: continue
    x, y = hcgen.config_inputs(cfg)
    xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    p = hc.Plan(D, str(x.dtype))
    z = torch.empty(3 ** D, dtype=xg.dtype, device="cuda")
    mn, md = t_ms(lambda: p.convolve(xg, yg, z), reps=3 if D >= 20 else 10)
    print(f"{name} D={D} {x.dtype}: min {mn:.3f} ms med {md:.3f} ms  ({z.numel()*8/mn/1e6:.0f} GB/s out)")
