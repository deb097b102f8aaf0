mkdir -p gpurun_out/n9
for lib in paper_1608_00206_b200/libhc.so variants/libhc_ep8.so variants/libhc_ep32.so; do for v in evalpoint evalpoint-peer; do
  echo "$lib $v k5: $(HC_LIB=$lib timeout 600 python bench.py --variant $v --ep-k 5 --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')"
done; done > gpurun_out/n9/t.txt
echo "k4: $(timeout 600 python bench.py --variant evalpoint --ep-k 4 --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')" >> gpurun_out/n9/t.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "evalpoint" 2>&1 | tail -1 >> gpurun_out/n9/t.txt
cat gpurun_out/n9/t.txt
