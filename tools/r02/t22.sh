for rep in 1 2; do for lib in paper_1608_00206_b200/libhc.so variants/libhc_minb3.so; do
  echo "$lib: $(HC_LIB=$lib timeout 200 python tools/quick_time.py c2 | tr '\n' ' ')"
done; done
