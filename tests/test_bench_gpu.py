"""bench.py end to end on the GPU: the N = 1 JSON contract, and the N > 1 path (torchrun, two
ranks, output split, barrier + max-over-ranks timing) with gloo so both ranks can share the
single GPU this environment provides."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c3_d16_i64", "--steps", "3", "--warmup", "3",
                        "--e2e-steps", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] >= 3
    assert d["roofline"]["frac"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["d2h_bytes_per_step"] == 8 * 3 ** 16


def test_bench_two_ranks_share_one_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--workload", "c3_d16_i64", "--steps", "2", "--warmup", "3", "--no-e2e",
                        "--dist-backend", "gloo"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "output-split x2"


@pytest.mark.parametrize("args,parallelism", [
    (["--workload", "c3_d16_i64", "--variant", "evalpoint", "--ep-k", "2"], "evalpoint k=2 x2 (all-to-all)"),
    (["--workload", "c3_d16_i64", "--variant", "evalpoint-peer", "--ep-k", "2"], "evalpoint k=2 x2 (peer reads)"),
    (["--workload", "c5_d22_f64", "--steps", "1", "--no-cpu-baseline"],
     "8 output-split shards streamed through one buffer, 4 per rank x2"),
])
def test_bench_two_ranks_variants(args, parallelism):
    # the evaluation-point variant (exchange staged through host memory under gloo) and the
    # streamed D = 22 workload, two ranks on the one GPU
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--no-e2e", "--dist-backend", "gloo"] + args
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == parallelism
