#!/bin/bash
# time D=20 for each variant .so (and skip modes): bash tools/variants_c4.sh v1 v2 ...
for v in "$@"; do
  for s in 0 1 2; do
    echo "== $v skip=$s"; HC_LIB=variants/libhc_$v.so HC_DEBUG_SKIP=$s timeout 300 python tools/quick_time.py c4 2>&1 | tail -4
  done
done
