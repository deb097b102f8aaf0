mkdir -p gpurun_out/n2
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --workload c2_b65536_d8_i64"
$B > gpurun_out/n2/plain.txt 2>&1; echo "plain rc=$?"; tail -c 1500 gpurun_out/n2/plain.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"tile8n" -s 1 -c 1 -o /tmp/p_n2 $B > gpurun_out/n2/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/p_n2.ncu-rep > gpurun_out/n2/summary.txt 2>&1
python tools/src_stalls.py /tmp/p_n2.ncu-rep 40 > gpurun_out/n2/stalls.txt 2>&1
python tools/smem_wavefronts.py /tmp/p_n2.ncu-rep 25 > gpurun_out/n2/smem.txt 2>&1
cat gpurun_out/n2/summary.txt
