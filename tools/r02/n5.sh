mkdir -p gpurun_out/n5
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "narrow or batched or c2 or HC_NARROW" > gpurun_out/n5/pt.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n5/pt.txt
for m in 2 1 2 1; do echo "HC_NARROW=$m"; HC_NARROW=$m timeout 120 python tools/quick_time.py c2; done
