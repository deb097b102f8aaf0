for rep in 1 2; do for ps in 1 0; do
  echo "pair_split=$ps: $(HC_PAIR_SPLIT=$ps timeout 300 python bench.py --workload c1_d10_i64 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep -o '"ms_per_step": [0-9.]*\|"launch_ms": [0-9.]*' | tr '\n' ' ')"
done; done
