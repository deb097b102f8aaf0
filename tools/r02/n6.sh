for rep in 1 2; do
for lib in paper_1608_00206_b200/libhc.so variants/libhc_instep.so; do for m in 1 2; do
  echo "$lib HC_NARROW=$m: $(HC_LIB=$lib HC_NARROW=$m timeout 120 python tools/quick_time.py c2 | tail -1)"
done; done; done
