#!/bin/bash
CMD="python tools/quick_time.py c4"
HC_DEBUG_SKIP=1 $CMD > gpurun_out/plain_p1.log 2>&1 && HC_DEBUG_SKIP=1 ncu --set full --clock-control none --import-source on -k regex:slab8 -s 2 -c 1 -o gpurun_out/prof_s8_p1 $CMD > gpurun_out/ncu_s8_p1.log 2>&1; echo rc=$?
$CMD > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:slab8 -s 2 -c 1 -o gpurun_out/prof_s8_full $CMD > gpurun_out/ncu_s8_full.log 2>&1; echo rc=$?
