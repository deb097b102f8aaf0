mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "narrow or batched or c2 or HC_NARROW" > gpurun_out/n1_pt.txt 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/n1_pt.txt
timeout 120 python tools/quick_time.py c2 > gpurun_out/n1_qt.txt 2>&1; echo "qt rc=$?"; cat gpurun_out/n1_qt.txt
HC_NARROW=0 timeout 120 python tools/quick_time.py c2; echo "qt0 rc=$?"
