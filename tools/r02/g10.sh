CMD="python tools/r02/sxprof.py 20"
for cfg in "HC_P2_HEAD=-1" "HC_P2_HEAD=0" "HC_P2_HEAD=243" "HC_P2_HEAD=486" "HC_P2_HEAD=243 HC_SLAB_LAG=2" "HC_P2_HEAD=0 HC_SLAB_LAG=2"; do
  echo "== $cfg"; env $cfg timeout -s KILL 120 $CMD 2>&1 | tail -1
done
for cfg in "HC_P2_HEAD=243" "HC_P2_HEAD=0"; do env $cfg timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:slab8 -s 1 -c 1 $CMD 2>&1 | grep -E "dram__"; done
HC_P2_HEAD=243 timeout -s KILL 120 python tools/r02/sx_quick.py 2>&1 | tail -4
