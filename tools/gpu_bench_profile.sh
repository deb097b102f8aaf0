#!/bin/bash
# On the GPU box: bench line, launch list, one full ncu capture of the top kernel.
# usage: bash tools/gpu_bench_profile.sh <tag> [workload]
TAG=${1:-r01}
WL=${2:-c4_d20_f64}
mkdir -p gpurun_out
python bench.py --workload $WL --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
CMD="python bench.py --workload $WL --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch-list rc=$?"
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"slab8|tile8|tile_kernel" -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu-full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
