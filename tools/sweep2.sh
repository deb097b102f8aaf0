#!/bin/bash
python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for eng in 1 0; do
  echo "== HC_ENGINE=$eng"; HC_ENGINE=$eng python tools/quick_time.py
done
for d in 1 2; do echo "engine skip=$d: $(HC_DEBUG_SKIP=$d python tools/quick_time.py c4 | tail -1)"; done
