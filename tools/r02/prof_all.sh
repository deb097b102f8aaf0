# bench-kernel ncu captures of every workload's dominant kernel (one GPU); summaries are made
# on the box (the reports themselves are too large to bring back, except c4's)
mkdir -p gpurun_out/prof
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
run() {  # tag, bench args, kernel regex, launch skip, traffic key
  rm -f /tmp/p_$1.ncu-rep   # /tmp survives on a reused box: never summarise a stale report
  $B $2 > gpurun_out/prof/$1.plain 2>&1 && \
  timeout -s KILL 600 ncu -f --set full --clock-control none --import-source on -k regex:"$3" -s ${4:-0} -c 1 -o /tmp/p_$1 $B $2 > gpurun_out/prof/$1.ncu.log 2>&1
  echo "$1 rc=$?"
  python tools/ncu_summary.py /tmp/p_$1.ncu-rep > gpurun_out/prof/$1.summary.txt 2>&1
  python tools/src_stalls.py /tmp/p_$1.ncu-rep 40 > gpurun_out/prof/$1.stalls.txt 2>&1
  python tools/smem_wavefronts.py /tmp/p_$1.ncu-rep 25 > gpurun_out/prof/$1.smem.txt 2>&1
  ncu -i /tmp/p_$1.ncu-rep --page raw --csv > gpurun_out/prof/$1.raw.csv 2>/dev/null
  [ -n "$5" ] && python tools/ncu_traffic.py /tmp/p_$1.ncu-rep "$5" "$3" >> gpurun_out/prof/traffic.log 2>&1
  cp profiles/ncu_traffic.json gpurun_out/prof/ncu_traffic.json 2>/dev/null
}
run c4 "--workload c4_d20_f64" "slab8" 1 "c4_d20_f64|split|slab"
cp /tmp/p_c4.ncu-rep gpurun_out/prof/c4.ncu-rep
run c2 "--workload c2_b65536_d8_i64" "tile8n" 1 "c2_b65536_d8_i64|split|tile"
run c3 "--workload c3_d16_i64" "slab8" 1 "c3_d16_i64|split|slab"
run c5 "--workload c5_d22_f64" "slab8" 8 "c5_d22_f64|split|slab"
run f1 "--workload f1_conv1d_d20_i64" "slab8" 1 "f1_conv1d_d20_i64|conv1d|slab"
run f2 "--workload f2_maxconv_d20_f64" "slab8" 1 "f2_maxconv_d20_f64|maxconv|slab"
run f4 "--workload f4_difference_d20_f64" "slab8" 1 "f4_difference_d20_f64|difference|slab"
run ep "--workload c4_d20_f64 --variant evalpoint --ep-k 4" "slab8" 1 "c4_d20_f64|evalpoint|slab"
run epinv "--workload c4_d20_f64 --variant evalpoint --ep-k 4" "ep_top_inverse" 1
run c1 "--workload c1_d10_i64" "tile8" 1 "c1_d10_i64|split|tile"
run epp "--workload c4_d20_f64 --variant evalpoint-peer --ep-k 4" "slab8" 1 "c4_d20_f64|evalpoint-peer|slab"
export HC_ENGINE=slabx; run sx "--workload c4_d20_f64" "slabx" 1 "c4_d20_f64|split|slab|slabx"; unset HC_ENGINE
$B --workload c4_d20_f64 > gpurun_out/prof/ll.plain 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c4.csv $B --workload c4_d20_f64 > gpurun_out/prof/ll.log 2>&1
echo "launch list rc=$?"
du -sh gpurun_out
$B --workload c2_b65536_d8_i64 > gpurun_out/prof/ll2.plain 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2.csv $B --workload c2_b65536_d8_i64 > gpurun_out/prof/ll2.log 2>&1
echo "launch list c2 rc=$?"
