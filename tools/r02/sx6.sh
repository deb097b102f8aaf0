echo "== slabx parity+time"; HC_ENGINE=slabx timeout -s KILL 100 python tools/r02/sx_quick.py 2>&1 | tail -9
for LAG in 2 3; do echo "== slabx prof lag $LAG"; HC_ENGINE=slabx HC_SLABX_LAG=$LAG HC_LIB=variants/libhc_prof.so timeout -s KILL 60 python tools/r02/sxprof.py 2>&1 | tail -2; done
