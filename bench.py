#!/usr/bin/env python
"""Benchmark of the hypercube-convolution hot path (BASELINE.json metric).

One "step" = one full convolution z = x * y of the named workload through the library's
C ABI (hc_convolve / hc_convolve_sharded) with inputs resident in HBM.  Default workload
(N = 1): BASELINE.json config 4, D = 20 fp64, x, y Exponential(1)-normalized (seeded,
synthetic; hcgen).  With N > 1 GPUs (torchrun), the same D = 20 output is split into N
contiguous ranges (zero-communication split by top trits, PAPER.md 166-177): total work
fixed -> "scaling": "strong"; time = max over ranks.

Prints ONE JSON line on rank 0: the contract keys, `roofline` (min-bytes HBM efficiency of
the dominant kernel from in-library per-launch CUDA events, plus the 8.0 TB/s spec figure and
ncu's DRAM GB/s), `co_roofline` (fp64 instructions of the two-level engine against the
measured fp64 rate), `cpu_baseline` (the oracle on a bounded sample of output cells), `e2e`
(hc_convolve_host with pinned host buffers), `gpu_launches` and `clocks`.  Workloads smaller
than 2x L2 are timed step by step with an L2 flush in between.  `--workload` selects the
other BASELINE configs and the SURVEY §8(f) application rows (f1 conv1d, f2 p-norm
max-convolution, f4 differences); `--variant evalpoint[-peer]` the K5b split.
`--impl reference` times the oracle (Algorithm 1 in plain C, oracle/) on the host cores
instead; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hcgen  # noqa: E402

L2_BYTES = 126 * 1024 * 1024  # B200 L2
METRIC = "output entries/s and achieved HBM GB/s vs roofline, D=20 fp64, 1/2/4/8 B200"
UNIT = "output entries/s"

WORKLOADS = {
    "c4_d20_f64": dict(cfg="c4_d20_f64", D=20, desc="single pair D=20 fp64, Exp(1)-normalized (BASELINE config 4)"),
    "c3_d16_i64": dict(cfg="c3_d16_i64", D=16, desc="single pair D=16 int64 uniform [0,2^16) (BASELINE config 3)"),
    "c1_d10_i64": dict(cfg="c1_d10_i64", D=10, desc="single pair D=10 int64 uniform [0,9] (BASELINE config 1)"),
    "c5_d22_f64": dict(cfg="c5_d22_f64", D=22, desc="single pair D=22 fp64 Exp(1)-normalized, sharded (BASELINE config 5)"),
    "c2_b65536_d8_i64": dict(cfg="c2_b65536_d8_i64", D=8, B=65536,
                             desc="65536 independent pairs D=8 int64 uniform [0,255] (BASELINE config 2)"),
    # SURVEY.md §8(f) rows, on config-4-sized inputs (D = 20)
    "f1_conv1d_d20_i64": dict(cfg="c3_like_d20_i64", D=20, app="conv1d",
                              desc="f1: ordinary 1-D convolution of two length-2^20 int64 vectors (uniform [0,2^16)) "
                                   "= carry-free hypercube convolution + carries"),
    "f2_maxconv_d20_f64": dict(cfg="c4_d20_f64", D=20, app="maxconv",
                               desc="f2: p-norm max-convolution (p = 16) of the config-4 inputs"),
    "f4_difference_d20_f64": dict(cfg="c4_d20_f64", D=20, app="difference",
                                  desc="f4: PMF of X - Y for the config-4 Bernoulli-axis PMFs"),
}


def workload_inputs(w):
    """Seeded synthetic inputs of a workload (hcgen): BASELINE configs, or the f1 row's vectors."""
    if w["cfg"] == "c3_like_d20_i64":
        return (hcgen.uniform_int(1020, 0, 1 << 20, 0, (1 << 16) - 1),
                hcgen.uniform_int(1020, 1, 1 << 20, 0, (1 << 16) - 1))
    return hcgen.config_inputs(w["cfg"])


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def csrc_sha():
    """sha256 over the CUDA sources of libhc.so: a captured DRAM-traffic figure is only reused
    for the exact kernel code it was captured on."""
    import glob
    import hashlib
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_1608_00206_b200", "csrc", "*"))):
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def load_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    ncu --set full capture of this exact workload / variant / kernel on this exact source
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py); else (None, reason)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, "no capture"
    with open(p) as f:
        d = json.load(f)
    e = d.get(key)
    if not isinstance(e, dict):
        return None, f"no capture for {key}"
    if e.get("csrc_sha") != csrc_sha():
        return None, f"capture for {key} is of other kernel sources ({e.get('csrc_sha')})"
    return e.get("bytes_per_launch"), e.get("source")


# int32 lane-instructions per output entry of the int64 (wrapping uint64) engines, from the
# kernels' arithmetic: 64-bit add / sub = 2 instructions, multiply-add mod 2^64 = 5; pair loop per
# tile = 243 units x (27 mad + 38 add) + 81 x 16 row sums + 96 F1 lanes x 19 adds + 32 x 8
# (cf. the fp64 model below), x (4/3)^k direct-split pairs; interpolation 2/3 sub per output
# and axis.  Peak: the fma and alu pipes each issue one warp instruction per 2 clk per SM
# sub-partition (B300_MICROARCH.md "Pipe rates") = 128 int32 lanes/clk/SM x 148 SMs at the
# 1965 MHz max clock = 37.2 T/s (derived, not measured).
INT32_PEAK = 148 * 128 * 1.965e9


def int_ops_per_output(D, k_top, interp_axes, narrow=False):
    if narrow:  # batched D = 8 in the 32-bit ring (hc_tile8n.cuh): one instruction per add / mad
        pair = (243 * (27 + 38) + 81 * 16 + 96 * 19 + 32 * 8) / 6561.0
        return pair + (2.0 / 3.0) * interp_axes + 1.0  # + the sign extension of each output
    pair = (243 * (27 * 5 + 38 * 2) + 81 * 16 * 2 + 96 * 19 * 2 + 32 * 8 * 2) / 6561.0
    return pair * (4.0 / 3.0) ** k_top + (4.0 / 3.0) * interp_axes


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=5)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        # under-load median: samples at >= 50% of max
        mx = max(smax) if smax else None
        loaded = [s for s in sm if mx and s >= 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def reduce_max(vals, dist=None, device="cuda"):
    """Elementwise max over ranks (device time is reported as the slowest rank's)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(vals)
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample_rate(wl, budget_s=10.0, seed=99):
    """Time the oracle (as it stands) on a bounded random sample of output cells of the
    workload; returns (entries/s, cores, sample description, seconds)."""
    import oracle
    oracle.build()
    w = WORKLOADS[wl]
    D = w["D"]
    cores = oracle.max_threads()
    if "B" in w:
        x, y = workload_inputs(w)
        rng = np.random.default_rng(seed)
        nb = 256
        bs = rng.choice(x.shape[0], size=nb, replace=False)
        t0 = time.perf_counter()
        oracle.conv_batched(x[bs], y[bs])
        dt = time.perf_counter() - t0
        n = nb * 3 ** D
        return n / dt, cores, f"{nb} of {x.shape[0]} cubes, full Algorithm 1 each ({n} entries)", dt
    x, y = workload_inputs(w)
    rng = np.random.default_rng(seed)
    m = 3 ** D
    n = 20000
    total_n, total_t = 0, 0.0
    while True:
        ks = rng.integers(0, m, size=n, dtype=np.int64).astype(np.uint64)
        t0 = time.perf_counter()
        oracle.conv_cells(x, y, ks)
        dt = time.perf_counter() - t0
        total_n += n
        total_t += dt
        if total_t >= budget_s * 0.5 or n >= 1 << 26:
            break
        n = int(min(1 << 26, max(n * 2, n * (budget_s * 0.6 - total_t) / max(dt, 1e-3))))
    return total_n / total_t, cores, (f"{total_n} uniformly random output cells of D={D} (Algorithm 1 gather "
                                      f"form, avg (4/3)^{D} pairs per cell)"), total_t


def config_dict(wl, args, world, flush=None):
    """The `config` object of the JSON line; identical for the repo arm and --impl reference."""
    w = WORKLOADS[wl]
    D = w["D"]
    n_total = w.get("B", 1) * 3 ** D
    in_bytes = 2 * w.get("B", 1) * 2 ** D * 8
    if flush is None:
        flush = n_total * 8 + in_bytes < 2 * L2_BYTES
    return {
        "workload": wl, "desc": w["desc"], "D": D, "output_entries": n_total,
        "variant": w.get("app", args.variant),
        "parallelism": (f"evalpoint k={args.ep_k} x{world} (all-to-all)" if args.variant == "evalpoint"
                        else f"evalpoint k={args.ep_k} x{world} (peer reads)" if args.variant == "evalpoint-peer"
                        else (f"{args.vshards} output-split shards streamed through one buffer, "
                              f"{args.vshards // world} per rank x{world}" if wl == "c5_d22_f64"
                              else (f"output-split x{world}" if world > 1 else "single"))),
        "l2": ("L2 flushed between steps (%d MB write, untimed), each step timed alone" % (4 * L2_BYTES >> 20)
               if flush else
               "output (%.2f GB) > 2 x L2 (126 MB): every step streams the whole output" % (n_total * 8 / 1e9)),
        "min_bytes_per_step": n_total * 8 + in_bytes,
    }


def run_reference(args, rank, world):
    if rank != 0:
        return
    wl = args.workload
    rates = []
    desc = None
    cores = None
    for _ in range(args.warmup):
        oracle_sample_rate(wl, budget_s=1.0, seed=7)
    t_all = 0.0
    for s in range(args.steps):
        r, cores, desc, dt = oracle_sample_rate(wl, budget_s=args.ref_budget, seed=100 + s)
        rates.append(r)
        t_all += dt
    v = statistics.median(rates)
    w = WORKLOADS[wl]
    n_entries = (w.get("B", 1)) * 3 ** w["D"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * n_entries / v, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if "f64" in wl else "int64", "data": "synthetic",
        "config": config_dict(wl, args, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                         "cpu": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "oracle = Algorithm 1 (PAPER.md 40-60) in plain C, OpenMP over cells; ms_per_step extrapolated "
                "from the sampled rate to the whole output",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4_d20_f64", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=8.0, help="seconds of oracle work per reference step")
    ap.add_argument("--variant", default="split", choices=["split", "evalpoint", "evalpoint-peer"],
                    help="multi-GPU scheme: 'split' = zero-communication output split (default); "
                         "'evalpoint' = top-axis evaluation points per rank + all-to-all + top inverse "
                         "(BASELINE north_star (4)); 'evalpoint-peer' = the same with the exchange fused "
                         "into the top inverse as direct peer reads (SURVEY §8(f) f3)")
    ap.add_argument("--ep-k", type=int, default=4, help="top axes of the evalpoint variant")
    ap.add_argument("--vshards", type=int, default=8,
                    help="c5 (D=22, 251 GB of output): the output is computed as this many shards of the "
                         "zero-communication split, streamed through one reused device buffer; rank r of N "
                         "runs shards [r*V/N, (r+1)*V/N)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets several ranks share one GPU (testing the N > 1 path on one device)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_1608_00206_b200.hc as hc

    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local_rank % max(ndev, 1))
    dist = None
    dev = "cuda"
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
            dev = "cpu"

    wl = args.workload
    w = WORKLOADS[wl]
    D = w["D"]
    batched = "B" in w
    plan = None
    x_np, y_np = workload_inputs(w)
    tdt = torch.float64 if x_np.dtype == np.float64 else torch.int64
    xg = torch.from_numpy(x_np).cuda()
    yg = torch.from_numpy(y_np).cuda()
    stream = torch.cuda.current_stream()

    if batched:
        if world > 1:
            raise SystemExit("batched workload is single-GPU in this bench")
        B = w["B"]
        z = torch.empty((B, 3 ** D), dtype=tdt, device="cuda")
        n_local = B * 3 ** D
        n_total = n_local

        def step():
            hc.convolve_batched(xg, yg, z)
        in_bytes = 2 * B * 2 ** D * 8
        prof_name = "tile"
    elif "app" in w:
        if world > 1:
            raise SystemExit("application workloads are single-GPU in this bench")
        app_plan = hc.Plan(D, str(x_np.dtype))
        z = torch.empty(3 ** D, dtype=tdt, device="cuda")
        n_local = n_total = 3 ** D
        if w["app"] == "conv1d":
            out1 = torch.empty((2 << D) - 1, dtype=tdt, device="cuda")

            def step():  # hc_conv1d: int64 at D >= 13 fuses the carries into pass 2, tiles in z
                hc.conv1d(xg, yg, out1, plan=app_plan, z_work=z)
        elif w["app"] == "maxconv":
            def step():
                app_plan.maxconv_pnorm(xg, yg, z, 16.0)
        else:
            def step():
                app_plan.convolve_difference(xg, yg, z)
        in_bytes = 2 * 2 ** D * 8
        prof_name = "slab"
        plan = None  # no host-buffer e2e for the application rows
    elif args.variant in ("evalpoint", "evalpoint-peer"):
        ep = hc.EPPlan(D, args.ep_k, str(x_np.dtype), world, rank)
        nc = 3 ** (D - args.ep_k)
        w_ep = torch.empty((ep.e1 - ep.e0) * nc, dtype=tdt, device="cuda")
        z = torch.empty(3 ** args.ep_k * (ep.c1 - ep.c0), dtype=tdt, device="cuda")
        n_local = z.numel()
        n_total = 3 ** D
        xdist = dist if world > 1 else None
        if args.variant == "evalpoint":
            wt = torch.empty_like(z)

            def step():
                ep.local(xg, yg, w_ep)
                hc.ep_exchange(w_ep, wt, D, args.ep_k, rank, world, xdist)
                ep.finish(wt, z)
        else:
            w_all = hc.ep_peer_buffers(w_ep, rank, world, xdist)

            def step():
                ep.local(xg, yg, w_ep)
                if xdist is not None:  # every rank's w is complete before anyone reads it
                    torch.cuda.synchronize()
                    xdist.barrier()
                ep.finish_peer(w_all, z)
                if xdist is not None:  # ... and read before the next step overwrites it
                    torch.cuda.synchronize()
                    xdist.barrier()
        in_bytes = 2 * 2 ** D * 8
        prof_name = "slab"
        plan = None
    elif wl == "c5_d22_f64":
        V = args.vshards
        if V % world != 0:
            raise SystemExit("--vshards must be a multiple of the number of ranks")
        vplans = [hc.Plan(D, str(x_np.dtype), V, s) for s in range(rank * V // world, (rank + 1) * V // world)]
        sizes = [e - b for b, e in (p.shard_info() for p in vplans)]
        zbuf = torch.empty(max(sizes), dtype=tdt, device="cuda")
        n_local = sum(sizes)
        n_total = 3 ** D

        def step():
            for p, m in zip(vplans, sizes):
                p.convolve_sharded(xg, yg, zbuf[:m])
        in_bytes = 2 * 2 ** D * 8
        prof_name = "slab"
    else:
        plan = hc.Plan(D, str(x_np.dtype), world, rank)
        zb, ze = plan.shard_info()
        z = torch.empty(ze - zb, dtype=tdt, device="cuda")
        n_local = ze - zb
        n_total = 3 ** D

        def step():
            plan.convolve_sharded(xg, yg, z)
        in_bytes = 2 * 2 ** D * 8
        prof_name = "tile"

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    barrier()

    sampler = ClockSampler(local_rank % max(ndev, 1))
    sampler.start()
    time.sleep(0.3)
    hc.prof_reset()
    hc.prof_enable(True)
    l0 = hc.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    step_bytes = n_total * 8 + in_bytes
    flush = step_bytes < 2 * L2_BYTES  # the step's data would stay L2-resident across steps
    barrier()
    torch.cuda.synchronize()
    if flush:
        # small workloads: write a buffer of 4x the L2 size between steps (untimed) and time
        # each step alone with events; the flush (~80 us) also keeps the device busy while the
        # host enqueues the step, so the events see the step's device time
        fbuf = torch.empty(4 * L2_BYTES, dtype=torch.uint8, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            fbuf.fill_(1)
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        t_sum = sum(a.elapsed_time(b) for a, b in evs)
        del fbuf
    else:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = hc.launch_count() - l0
    hc.prof_enable(False)
    clocks = sampler.stop()
    t_ms = t_sum if flush else e0.elapsed_time(e1)
    ktime, kcount = hc.prof_read(prof_name)
    if kcount == 0:
        prof_name = "slab"
        ktime, kcount = hc.prof_read(prof_name)
    hc.prof_reset()

    t_max, k_avg = reduce_max([t_ms, ktime / max(kcount, 1)], dist, device=dev)
    ms_per_step = t_max / args.steps
    value = n_total / (ms_per_step / 1e3)

    # roofline of the dominant kernel: algorithmic bytes (or operations) per launch / avg launch time
    launches_per_step = kcount / max(args.steps, 1)
    lps = max(launches_per_step, 1)
    peak, peak_src = load_peaks()
    evalpoint = args.variant in ("evalpoint", "evalpoint-peer") and "app" not in w and not batched
    if evalpoint:
        # the dominant launch is the batch of the rank's (D-k)-dimensional convolutions, one per
        # owned evaluation point (slab engine over points x slabs)
        Dl = D - args.ep_k
        npts = (ep.e1 - ep.e0) / lps
        outs_per_launch = npts * 3 ** Dl
        alg_bytes_per_launch = float(npts * (3 ** Dl + 2 * 2 ** Dl) * 8)
    else:
        outs_per_launch = n_local / lps
        alg_bytes_per_launch = (n_local * 8 + in_bytes * lps) / lps
    achieved = alg_bytes_per_launch / (k_avg / 1e3) / 1e9 if k_avg > 0 else None
    tkey = f"{wl}|{w.get('app', args.variant)}|{prof_name}" + ("|slabx" if os.environ.get("HC_ENGINE") == "slabx" else "")
    traffic, tsrc = load_traffic(tkey)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_source": tsrc,
                "kernel": prof_name, "alg_bytes_per_launch": alg_bytes_per_launch, "launch_ms": k_avg,
                "launches_per_step": launches_per_step, "peak_source": peak_src,
                # the same efficiency against the 8.0 TB/s spec figure, and the
                # DRAM traffic ncu measured for this launch (profiles/ncu_traffic.json) over its time
                "frac_vs_spec_8000": (achieved / 8000.0) if achieved else None,
                "dram_gbs": (traffic / (k_avg / 1e3) / 1e9) if (traffic and k_avg > 0) else None}
    k_top = max(D - 14, 0) if D >= 13 else max(D - 8, 0)
    interp = min(D, 14) if D >= 13 else min(D, 8)
    if w.get("app") == "conv1d":
        # f1: the 1-D convolution's output is 2^(D+1) - 1 entries (16.8 MB at D = 20), so the 3^D
        # write is not in the algorithm; the fused kernel is bound by integer arithmetic
        ops = int_ops_per_output(D, k_top, interp) * 3 ** D / lps
        out_b = ((2 << D) - 1) * 8 + in_bytes
        roofline = {"bound": "alu", "achieved": ops / (k_avg / 1e3) / 1e12 if k_avg else None,
                    "peak": INT32_PEAK / 1e12, "unit": "T int32 lane-instr/s",
                    "frac": (ops / (k_avg / 1e3) / INT32_PEAK) if k_avg else None,
                    "ops_per_hypercube_output": int_ops_per_output(D, k_top, interp), "kernel": prof_name,
                    "launch_ms": k_avg, "peak_source": "derived: 128 int32 lanes/clk/SM x 148 SMs x 1965 MHz",
                    "traffic": traffic, "traffic_source": tsrc,
                    "hbm_min_bytes_frac": (out_b / (k_avg / 1e3) / 1e9 / peak) if k_avg else None}
    # fp64 co-roofline of the two-level engine (DESIGN.md §4 cost model): algorithmic fp64
    # instructions per output entry = pair loop (F2 27 FMA + 38 add per unit and pair, 16 row
    # sums on the e_a2 = 1 units, F1 19 adds (+8) per lane) x (4/3)^k pairs + 2/3 per
    # interpolated axis (tile and middle axes); against the measured DADD/DFMA lane rate.
    # int64 workloads: the int32-instruction model above against the derived INT peak.
    co = None
    Dk = D - args.ep_k if evalpoint else D
    ktop_k = (max(Dk - 14, 0) if Dk >= 13 else max(Dk - 8, 0))
    interp_k = min(Dk, 14) if Dk >= 13 else min(Dk, 8)
    if tdt == torch.float64 and w.get("app") != "conv1d":
        pair_ops = (243 * (27 + 38) + 81 * 16 + 96 * 19 + 32 * 8) / 6561.0
        ops_per_out = pair_ops * (4.0 / 3.0) ** ktop_k + (2.0 / 3.0) * interp_k
        ops = ops_per_out * outs_per_launch
        fp64_peak = 17.5e12  # fp64 lane-instructions/s measured on this B200 (DFMA 17.0, DADD 18.5 T/s)
        co = {"bound": "fp64", "ops_per_output": ops_per_out, "achieved": ops / (k_avg / 1e3) / 1e12 if k_avg else None,
              "peak": fp64_peak / 1e12, "unit": "T fp64 instr-lanes/s",
              "frac": (ops / (k_avg / 1e3) / fp64_peak) if k_avg else None}
    elif tdt == torch.int64 and w.get("app") != "conv1d":
        narrow = batched and D == 8 and os.environ.get("HC_NARROW", "1") != "0"
        ops_per_out = int_ops_per_output(Dk, ktop_k, interp_k, narrow)
        ops = ops_per_out * outs_per_launch
        co = {"bound": "int", "ops_per_output": ops_per_out,
              "achieved": ops / (k_avg / 1e3) / 1e12 if k_avg else None, "peak": INT32_PEAK / 1e12,
              "unit": "T int32 lane-instr/s", "frac": (ops / (k_avg / 1e3) / INT32_PEAK) if k_avg else None,
              "peak_source": "derived: 128 int32 lanes/clk/SM x 148 SMs x 1965 MHz"}

    # end to end through the host-buffer C-ABI entry point (pinned host memory, copies inside)
    e2e = None
    if not args.no_e2e and not batched and plan is not None:
        xh = torch.from_numpy(x_np).pin_memory()
        yh = torch.from_numpy(y_np).pin_memory()
        zh = torch.empty(n_local, dtype=tdt).pin_memory()
        plan.convolve_host(xh, yh, zh)  # warm (allocates the plan's device workspace)
        barrier()
        ts = []
        for _ in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            plan.convolve_host(xh, yh, zh)
            ts.append(time.perf_counter() - t0)
        tm = reduce_max([statistics.median(ts)], dist, device=dev)[0]
        e2e = {"value": n_total / tm, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
               "d2h_bytes_per_step": n_total * 8, "seconds_per_step": tm,
               "path": "hc_convolve_host (pinned host x,y -> device -> pinned host z, chunked D2H overlapped)"}
        del zh
    elif not args.no_e2e and batched:
        # batched: the caller's sequence with the public binding -- pinned host x, y -> device,
        # hc_convolve_batched, device z -> pinned host, all on the current stream, synchronised
        xh = torch.from_numpy(x_np).pin_memory()
        yh = torch.from_numpy(y_np).pin_memory()
        zh = torch.empty(tuple(z.shape), dtype=tdt).pin_memory()

        def e2e_step():
            xg.copy_(xh, non_blocking=True)
            yg.copy_(yh, non_blocking=True)
            hc.convolve_batched(xg, yg, z)
            zh.copy_(z, non_blocking=True)
            torch.cuda.synchronize()
        e2e_step()
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t0)
        tm = statistics.median(ts)
        e2e = {"value": n_total / tm, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
               "d2h_bytes_per_step": n_total * 8, "seconds_per_step": tm,
               "path": "pinned host x,y -> device (torch copy), hc_convolve_batched, device z -> pinned host"}
        del zh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, cores, desc, dt = oracle_sample_rate(wl, budget_s=10.0)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, "seconds": dt,
               "cpu": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if tdt == torch.float64 else "int64",
            "data": "synthetic",
            "config": config_dict(wl, args, world, flush),
            "hbm_gbs_min_bytes": (n_total * 8 + in_bytes) / (ms_per_step / 1e3) / 1e9,
            "roofline": roofline, "co_roofline": co, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
