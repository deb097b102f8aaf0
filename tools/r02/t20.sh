# re-sweep of the slab-engine knobs with the 2-stage ring
for rep in 1 2; do
  echo "base: $(timeout 200 python tools/quick_time.py c4 c3 | tr '\n' ' ')"
  echo "lag2: $(HC_SLAB_LAG=2 timeout 200 python tools/quick_time.py c4 c3 | tr '\n' ' ')"
  echo "p2ch1: $(HC_LIB=variants/libhc_p2ch1.so timeout 200 python tools/quick_time.py c4 c3 | tr '\n' ' ')"
done
for lib in paper_1608_00206_b200/libhc.so variants/libhc_epi2.so; do
  echo "$lib f1: $(HC_LIB=$lib timeout 600 python bench.py --workload f1_conv1d_d20_i64 --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')"
done
