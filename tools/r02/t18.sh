for rep in 1 2; do for lib in paper_1608_00206_b200/libhc.so variants/libhc_rowmajor.so; do
  echo "$lib: $(HC_LIB=$lib timeout 120 python tools/quick_time.py c2 | tail -1)"
done; done
HC_LIB=variants/libhc_rowmajor.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "narrow or c2" 2>&1 | tail -1
