# the driver's default command, three times back to back (run-to-run spread of the headline)
for i in 1 2 3; do
  t0=$(date +%s.%N); timeout 900 python bench.py > gpurun_out/rep_$i.json 2> gpurun_out/rep_$i.err; rc=$?; t1=$(date +%s.%N)
  echo "run $i rc=$rc wall $(python -c "print(round($t1-$t0,1))") s: $(grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"sm_mhz": [0-9.]*' gpurun_out/rep_$i.json | head -3 | tr '\n' ' ')"
done
