# copy a finalisation pass (fin*.sh) from gpurun_out/ into profiles/r02/ and profiles/ncu_traffic.json
R=profiles/r02
for wl in c1_d10_i64 c2_b65536_d8_i64 c3_d16_i64 c4_d20_f64 c5_d22_f64 f1_conv1d_d20_i64 f2_maxconv_d20_f64 f4_difference_d20_f64; do cp gpurun_out/b_$wl.json $R/bench_$wl.json; done
for v in ep epp slabx ref; do cp gpurun_out/b_$v.json $R/bench_$v.json; done
for t in c1 c2 c3 c4 c5 f1 f2 f4 ep epp epinv sx; do (cat gpurun_out/prof/$t.summary.txt; cat gpurun_out/prof/$t.smem.txt) > $R/ncu_$t.txt; cp gpurun_out/prof/$t.stalls.txt $R/ncu_${t}_src_stalls.txt; done
python tools/launch_list.py gpurun_out/prof/launches_c4.csv "ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --workload c4_d20_f64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline (cold-cache, serialised launches)" > $R/launch_list_c4_d20.txt
python tools/launch_list.py gpurun_out/prof/launches_c2.csv "ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --workload c2_b65536_d8_i64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline (cold-cache, serialised launches)" > $R/launch_list_c2_b65536_d8.txt
cp gpurun_out/$1_tests.txt $R/gpu_tests_final.txt
cp gpurun_out/prof/ncu_traffic.json profiles/ncu_traffic.json
