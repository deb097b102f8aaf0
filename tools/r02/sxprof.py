"""One D=20 convolution with the phase-profiling build (HC_LIB=variants/libhc_prof.so)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import hcgen
import paper_1608_00206_b200.hc as hc
D = int(sys.argv[1]) if len(sys.argv) > 1 else 20
x, y = hcgen.config_inputs('c4_d20_f64') if D == 20 else hcgen.make_pair(D, 'float64', 'exp_norm', 7)
xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
p = hc.Plan(D, 'float64')
z = torch.empty(3 ** D, dtype=torch.float64, device='cuda')
for i in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p.convolve(xg, yg, z); e1.record(); torch.cuda.synchronize()
    print(f"run {i}: {e0.elapsed_time(e1):.2f} ms", flush=True)
