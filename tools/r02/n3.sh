mkdir -p gpurun_out/n3
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "narrow or batched or c2" > gpurun_out/n3/pt.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/n3/pt.txt
timeout 120 python tools/quick_time.py c2; echo "qt rc=$?"
timeout 120 python bench.py --workload c2_b65536_d8_i64 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/n3/bench.txt 2>&1; echo "bench rc=$?"; tail -c 1200 gpurun_out/n3/bench.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n3/ll.csv python tools/quick_time.py c2 > /dev/null 2>&1; echo "ll rc=$?"
grep -o '"[a-zA-Z_:<>0-9 ]*kernel[^"]*","[^"]*","gpu__time_duration.sum","[^"]*","[0-9.]*"' gpurun_out/n3/ll.csv | tail -8
tail -8 gpurun_out/n3/ll.csv | cut -c1-300
