mkdir -p gpurun_out/n8
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "evalpoint" > gpurun_out/n8/pt.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/n8/pt.txt
for k in 4 5; do for v in evalpoint evalpoint-peer; do
  timeout 600 python bench.py --variant $v --ep-k $k --no-cpu-baseline > gpurun_out/n8/b_${v}_k$k.json 2> gpurun_out/n8/b_${v}_k$k.err; echo "$v k=$k rc=$?"
  grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"launch_ms": [0-9.]*' gpurun_out/n8/b_${v}_k$k.json | tr '\n' ' '; echo
done; done
timeout 300 python bench.py --workload c2_b65536_d8_i64 --no-cpu-baseline > gpurun_out/n8/b_c2.json 2>&1; echo "c2 rc=$?"; grep -o '"e2e": {[^}]*}' gpurun_out/n8/b_c2.json
