mkdir -p gpurun_out
nvidia-smi > gpurun_out/g1_smi.txt 2>&1
timeout 120 ./tools/microbench/mb10 > gpurun_out/g1_mb10.txt 2>&1; echo "mb10 rc=$?"
cat gpurun_out/g1_mb10.txt
timeout 300 python tools/quick_time.py c2 c3 c1 c4 > gpurun_out/g1_qt.txt 2>&1; echo "qt rc=$?"
cat gpurun_out/g1_qt.txt
