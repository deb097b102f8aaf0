# bench lines of every workload (one GPU); JSON lines to gpurun_out/b_<workload>.json
mkdir -p gpurun_out
for wl in c4_d20_f64 c2_b65536_d8_i64 c3_d16_i64 c1_d10_i64 f1_conv1d_d20_i64 f2_maxconv_d20_f64 f4_difference_d20_f64; do
  timeout -s KILL 600 python bench.py --workload $wl > gpurun_out/b_$wl.json 2> gpurun_out/b_$wl.err; echo "$wl rc=$?"
done
timeout -s KILL 900 python bench.py --workload c5_d22_f64 --steps 3 --warmup 3 > gpurun_out/b_c5_d22_f64.json 2> gpurun_out/b_c5.err; echo "c5 rc=$?"
timeout -s KILL 600 python bench.py --variant evalpoint --ep-k 4 > gpurun_out/b_ep.json 2> gpurun_out/b_ep.err; echo "ep rc=$?"
timeout -s KILL 600 python bench.py --variant evalpoint-peer --ep-k 4 > gpurun_out/b_epp.json 2> gpurun_out/b_epp.err; echo "epp rc=$?"
HC_ENGINE=slabx timeout -s KILL 600 python bench.py --workload c4_d20_f64 --no-cpu-baseline > gpurun_out/b_slabx.json 2> gpurun_out/b_slabx.err; echo "slabx rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo "ref rc=$?"
