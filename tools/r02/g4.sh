for L in 5 6 7 8; do echo "== L'=$L"; HC_SMALL_L=$L timeout -s KILL 120 python tools/r02/small.py 2>&1 | tail -4; done
