timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "two_level or geometr or shard or D13 or d13 or 13" 2>&1 | tail -2
timeout 300 python tools/r02/t14.py 2>&1 | grep "D=1[3-7]"
