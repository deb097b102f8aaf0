for LAG in 1 2 3; do echo "== lag $LAG"; HC_SLABX_LAG=$LAG HC_LIB=variants/libhc_prof.so timeout -s KILL 120 python tools/r02/sxprof.py 2>&1 | tail -2; done
echo "== slab8 prof"; HC_ENGINE=slab8 HC_LIB=variants/libhc_prof.so timeout -s KILL 120 python tools/r02/sxprof.py 2>&1 | tail -2
