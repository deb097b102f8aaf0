#!/bin/bash
# timing experiments for the slab engine (not bench numbers)
for s in 14 13; do
  for d in 0 1 2; do
    echo "slab_axes=$s skip=$d: $(HC_SLAB_AXES=$s HC_DEBUG_SKIP=$d python tools/quick_time.py c4 | tail -1)"
  done
done
