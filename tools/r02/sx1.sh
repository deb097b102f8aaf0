mkdir -p gpurun_out
echo "== slabx"; timeout -s KILL 300 python tools/r02/sx_quick.py 2>&1 | tail -12
echo "== slab8"; HC_ENGINE=slab8 timeout -s KILL 300 python tools/r02/sx_quick.py 2>&1 | tail -4
