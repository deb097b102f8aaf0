"""Balance of the zero-communication output split (K5a; PAPER.md 166-177), measured
on ONE B200: every shard of an N-way split is run alone (hc_convolve_sharded) and timed with CUDA
events.  max/mean over the shards is the split's scaling ceiling on N GPUs (no collective on the
data path).  Also fits the slab cost model t = a * (#slabs) + b * (sum of 2^{#1(t_T)}) by least
squares over all shards and prints alpha = a / b (the constant of compute_cuts, hc_api.cu).
usage: python tools/shard_times.py [D ...]   (env HC_SHARD_ALPHA selects the cut model)"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hcgen
import paper_1608_00206_b200.hc as hc

def ones_count(t, k):
    c = 0
    for _ in range(k):
        c += t % 3 == 1
        t //= 3
    return c

rows = []
out = {"alpha_env": os.environ.get("HC_SHARD_ALPHA"), "runs": []}
for D in [int(a) for a in sys.argv[1:]] or [20, 22]:
    x, y = hcgen.config_inputs("c4_d20_f64" if D == 20 else "c5_d22_f64")
    xg, yg = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    k = D - 14
    unit = 3 ** 14
    for N in (2, 4, 8):
        times, feats = [], []
        zbuf = None
        for r in range(N):
            p = hc.Plan(D, "float64", N, r)
            b, e = p.shard_info()
            n = e - b
            if zbuf is None or zbuf.numel() < n:
                zbuf = None
                torch.cuda.empty_cache()
                zbuf = torch.empty(n, dtype=torch.float64, device="cuda")
            zs = zbuf[:n]
            p.convolve_sharded(xg, yg, zs)
            torch.cuda.synchronize()
            ts = []
            for _ in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); p.convolve_sharded(xg, yg, zs); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = min(ts)
            s0, s1 = b // unit, e // unit
            pairs = sum(1 << ones_count(t_, k) for t_ in range(s0, s1))
            times.append(t)
            feats.append((s1 - s0, pairs))
            del p, zs
        mx, mean = max(times), sum(times) / N
        run = {"D": D, "N": N, "shard_ms": [round(t, 3) for t in times], "max_over_mean": mx / mean,
               "sum_ms": sum(times), "speedup_ceiling": sum(times) / mx, "slabs_pairs": feats}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
        rows += [(f[0], f[1], t) for f, t in zip(feats, times)]
        del zbuf
        torch.cuda.empty_cache()
A = np.array([[r[0], r[1]] for r in rows], dtype=float)
t = np.array([r[2] for r in rows])
(a, bcoef), *_ = np.linalg.lstsq(A, t, rcond=None)
out["fit_ms_per_slab"] = a
out["fit_ms_per_pair_slab"] = bcoef
out["alpha_fit"] = a / bcoef
print(json.dumps({"fit": {"ms_per_slab": a, "ms_per_pair_slab": bcoef, "alpha": a / bcoef}}), flush=True)
