CMD="python tools/r02/sxprof.py 20"
for cfg in "HC_KEEP_POLICY=0" "HC_KEEP_POLICY=1" "HC_KEEP_POLICY=2" "HC_KEEP_POLICY=0 HC_L2_PERSIST_MB=96" "HC_KEEP_POLICY=0 HC_L2_PERSIST_MB=120"; do
  echo "== $cfg"; env $cfg timeout -s KILL 120 $CMD 2>&1 | tail -1
  env $cfg timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:slab8 -s 1 -c 1 $CMD 2>&1 | grep -E "dram__"
done
