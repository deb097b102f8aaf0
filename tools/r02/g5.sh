mkdir -p gpurun_out
for S in 14 13; do for LAG in 1 2; do echo "== slab axes $S lag $LAG"; HC_SLAB_AXES=$S HC_SLAB_LAG=$LAG timeout -s KILL 120 python tools/r02/sxprof.py 20 2>&1 | tail -1; done; done
CMD="python tools/r02/sxprof.py 20"
HC_SLAB_AXES=13 $CMD > /dev/null 2>&1 && HC_SLAB_AXES=13 timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct -k regex:slab8 -s 1 -c 1 $CMD 2>&1 | grep -E "dram__|gpu__time|hit_rate"
