#!/bin/bash
# On the GPU box: re-run every bench line kept under profiles/ (round tag $1).
TAG=${1:-r01}
mkdir -p gpurun_out
run() {  # name, args...
  local name=$1; shift
  python bench.py "$@" > gpurun_out/${TAG}_bench_$name.json 2> gpurun_out/${TAG}_bench_$name.err
  echo "$name rc=$? $(python -c "import json,sys;d=json.load(open('gpurun_out/${TAG}_bench_$name.json'));print(d['ms_per_step'],'ms', d.get('roofline',{}) and d['roofline'].get('frac'))" 2>&1)"
}
run c1_d10 --workload c1_d10_i64
run c2_b65536_d8 --workload c2_b65536_d8_i64
run c3_d16 --workload c3_d16_i64
run c5_d22_streamed --workload c5_d22_f64 --steps 3 --warmup 3
run c4_d20_evalpoint_k4 --workload c4_d20_f64 --variant evalpoint --steps 5
run c4_d20_evalpoint_peer_k4 --workload c4_d20_f64 --variant evalpoint-peer --steps 5
run f4_difference_d20_f64 --workload f4_difference_d20_f64 --steps 5
run f1_conv1d_d20_i64 --workload f1_conv1d_d20_i64 --steps 3
run f2_maxconv_d20_f64 --workload f2_maxconv_d20_f64 --steps 3
run c4_d20 --workload c4_d20_f64 --steps 10
