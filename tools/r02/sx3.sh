CMD="python tools/r02/sxprof.py 20"
HC_SLABX_LAG=3 timeout -s KILL 120 $CMD > gpurun_out/sx3_plain.log 2>&1 && \
HC_SLABX_LAG=3 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:slabx -s 1 -c 1 -o gpurun_out/sx3 $CMD > gpurun_out/sx3_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/sx3_ncu.log
