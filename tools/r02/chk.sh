# the whole GPU suite against the bounds-checked build (device asserts on every engine's index invariants)
mkdir -p gpurun_out
HC_LIB=variants/libhc_check.so timeout 3000 python -m pytest tests -m gpu -x -q -rs > gpurun_out/chk_tests.txt 2>&1; echo "check-build tests rc=$?"; tail -4 gpurun_out/chk_tests.txt
HC_LIB=variants/libhc_check.so timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"ms_per_step": [0-9.]*'
