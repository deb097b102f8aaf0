"""Development aid: fused conv1d timing, tiles in the plan's ring vs in place in a 3^D z_work."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import hcgen
import paper_1608_00206_b200.hc as hc
D = int(sys.argv[1]) if len(sys.argv) > 1 else 20
x = torch.from_numpy(hcgen.uniform_int(1020, 0, 1 << D, 0, (1 << 16) - 1)).cuda()
y = torch.from_numpy(hcgen.uniform_int(1020, 1, 1 << D, 0, (1 << 16) - 1)).cuda()
p = hc.Plan(D, "int64")
out = torch.empty((2 << D) - 1, dtype=torch.int64, device="cuda")
zw = torch.empty(3 ** D, dtype=torch.int64, device="cuda")
for name, kw in (("in place", {"z_work": zw}), ("ring", {})):
    try:
        for _ in range(2):
            hc.conv1d(x, y, out, plan=p, **kw)
    except hc.HCError as e:
        print(f"D={D} {name}: {e}")
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        hc.conv1d(x, y, out, plan=p, **kw)
    e1.record()
    torch.cuda.synchronize()
    print(f"D={D} {name}: {e0.elapsed_time(e1) / 3:.2f} ms")
