#!/bin/bash
CMD="python tools/quick_time.py c4"
HC_DEBUG_SKIP=1 $CMD > gpurun_out/plain_p1.log 2>&1 && HC_DEBUG_SKIP=1 ncu --set full --clock-control none --import-source on -k regex:engine -s 2 -c 1 -o gpurun_out/prof_eng_p1 $CMD > gpurun_out/ncu_eng_p1.log 2>&1; echo rc=$?
