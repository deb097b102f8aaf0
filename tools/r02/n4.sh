# EP batched points, f1 without spills: parity + timing
mkdir -p gpurun_out/n4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "evalpoint or conv1d or carries or narrow or variants" > gpurun_out/n4/pt.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/n4/pt.txt
for v in evalpoint evalpoint-peer; do
  timeout 600 python bench.py --variant $v --ep-k 4 --no-cpu-baseline > gpurun_out/n4/b_$v.json 2> gpurun_out/n4/b_$v.err; echo "$v rc=$?"
  grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"launch_ms": [0-9.]*\|"gpu_launches": [0-9]*' gpurun_out/n4/b_$v.json | tr '\n' ' '; echo
done
timeout 600 python bench.py --workload f1_conv1d_d20_i64 --no-cpu-baseline > gpurun_out/n4/b_f1.json 2> gpurun_out/n4/b_f1.err; echo "f1 rc=$?"
grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*' gpurun_out/n4/b_f1.json | tr '\n' ' '; echo
