for o in cost gray; do for tp in 0 1 2; do
  echo "order=$o table_policy=$tp: $(HC_SLAB_ORDER=$o HC_TABLE_POLICY=$tp timeout 200 python tools/quick_time.py c4 | tail -1)"
done; done
for o in cost gray; do for tp in 0 1; do
  HC_SLAB_ORDER=$o HC_TABLE_POLICY=$tp timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:slab8 -s 1 -c 1 python tools/quick_time.py c4 2>&1 | grep -E "dram__" | sed "s|^|$o/$tp |"
done; done
