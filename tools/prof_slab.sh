#!/bin/bash
# On the GPU box: one full ncu capture of the D=20 slab kernel (after a clean run).
TAG=${1:-dev}
CMD="python tools/quick_time.py c4"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:slab8 -s 2 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_$TAG.log
