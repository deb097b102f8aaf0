for S in 14 13; do echo "== slab axes $S"; HC_SLAB_AXES=$S timeout -s KILL 100 python tools/quick_time.py c3 2>&1 | tail -1; done
