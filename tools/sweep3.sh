#!/bin/bash
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
echo "== engine"; timeout 300 python tools/quick_time.py
for d in 1 2; do echo "engine skip=$d: $(HC_DEBUG_SKIP=$d timeout 120 python tools/quick_time.py c4 | tail -1)"; done
