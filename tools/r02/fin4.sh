# captures + bench lines of the evalpoint-peer and slabx variants under their own traffic keys
mkdir -p gpurun_out/prof
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
run() {
  rm -f /tmp/p_$1.ncu-rep
  $B $2 > gpurun_out/prof/$1.plain 2>&1 && \
  timeout -s KILL 600 ncu -f --set full --clock-control none --import-source on -k regex:"$3" -s ${4:-0} -c 1 -o /tmp/p_$1 $B $2 > gpurun_out/prof/$1.ncu.log 2>&1
  echo "$1 rc=$?"
  python tools/ncu_summary.py /tmp/p_$1.ncu-rep > gpurun_out/prof/$1.summary.txt 2>&1
  python tools/src_stalls.py /tmp/p_$1.ncu-rep 40 > gpurun_out/prof/$1.stalls.txt 2>&1
  python tools/smem_wavefronts.py /tmp/p_$1.ncu-rep 25 > gpurun_out/prof/$1.smem.txt 2>&1
  [ -n "$5" ] && python tools/ncu_traffic.py /tmp/p_$1.ncu-rep "$5" "$3" >> gpurun_out/prof/traffic.log 2>&1
  cp profiles/ncu_traffic.json gpurun_out/prof/ncu_traffic.json
}
run epp "--workload c4_d20_f64 --variant evalpoint-peer --ep-k 4" "slab8" 1 "c4_d20_f64|evalpoint-peer|slab"
export HC_ENGINE=slabx; run sx "--workload c4_d20_f64" "slabx" 1 "c4_d20_f64|split|slab|slabx"; unset HC_ENGINE
timeout -s KILL 600 python bench.py --variant evalpoint-peer --ep-k 4 > gpurun_out/b_epp.json 2> gpurun_out/b_epp.err; echo "epp rc=$?"
HC_ENGINE=slabx timeout -s KILL 600 python bench.py --workload c4_d20_f64 --no-cpu-baseline > gpurun_out/b_slabx.json 2> gpurun_out/b_slabx.err; echo "slabx rc=$?"
timeout -s KILL 600 python bench.py --workload c2_b65536_d8_i64 > gpurun_out/b_c2_b65536_d8_i64.json 2> gpurun_out/b_c2.err; echo "c2 rc=$?"
