# full GPU test suite incl. the D=20 full-output parity tests
mkdir -p gpurun_out
nproc > gpurun_out/g2_nproc.txt
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/g2_tests.txt 2>&1
echo "tests rc=$?"
tail -30 gpurun_out/g2_tests.txt
