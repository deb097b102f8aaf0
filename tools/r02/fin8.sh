# round-2 finalisation pass: full GPU suite, ncu captures of every workload, bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/fin8_tests.txt 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/fin8_tests.txt
bash tools/r02/prof_all.sh
bash tools/r02/bench_all.sh
