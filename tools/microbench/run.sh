#!/bin/bash
# run on the GPU box: bash tools/microbench/run.sh
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > ../../gpurun_out/mb_clocks.csv &
SMI=$!
./mb > ../../gpurun_out/mb.txt 2>&1
RC=$?
kill $SMI
cat ../../gpurun_out/mb.txt
exit $RC
