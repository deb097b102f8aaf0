for v in nraw6 nraw8 p2ch1; do echo "== $v"; HC_LIB=variants/libhc_$v.so timeout -s KILL 120 python tools/r02/sxprof.py 20 2>&1 | tail -1; done
echo "== default"; timeout -s KILL 120 python tools/r02/sxprof.py 20 2>&1 | tail -1
