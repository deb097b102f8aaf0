for lib in paper_1608_00206_b200/libhc.so variants/libhc_ep5c25.so variants/libhc_ep5c40.so variants/libhc_ep5c60.so; do
  echo "$lib k5: $(HC_LIB=$lib timeout 600 python bench.py --variant evalpoint --ep-k 5 --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')"
done
