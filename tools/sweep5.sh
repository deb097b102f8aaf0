#!/bin/bash
timeout 200 python -m pytest tests -x -q -m gpu -k "c4 or c3 or sharded" 2>&1 | tail -2
for lag in 1 2 3; do echo "lag=$lag: $(HC_SLAB_LAG=$lag timeout 120 python tools/quick_time.py c4 | tail -1)"; done
for lag in 1 2; do echo "s13 lag=$lag: $(HC_SLAB_AXES=13 HC_SLAB_LAG=$lag timeout 120 python tools/quick_time.py c4 | tail -1)"; done
