timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "single_pair_all_D or c1 or wraparound or sharded or host_entry or delta or variants" 2>&1 | tail -2
echo "== pair split"; timeout 300 python tools/r02/t25.py
echo "== per tile"; HC_PAIR_SPLIT=0 timeout 300 python tools/r02/t25.py
