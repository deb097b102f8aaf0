#!/bin/bash
CMD="python tools/quick_time.py c4"
$CMD > gpurun_out/plain_eng.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:engine -s 2 -c 1 -o gpurun_out/prof_eng_full $CMD > gpurun_out/ncu_eng_full.log 2>&1; echo rc=$?
