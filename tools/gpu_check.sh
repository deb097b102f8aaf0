#!/bin/bash
# On the GPU box: GPU parity tests, then quick device timings of the hot configs.
# usage: bash tools/gpu_check.sh <tag> [configs...]
TAG=${1:-dev}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.txt 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests_$TAG.txt
timeout 600 python tools/quick_time.py ${@:-c2 c3 c1 c4} > gpurun_out/qt_$TAG.txt 2>&1
echo "qt rc=$?"; cat gpurun_out/qt_$TAG.txt
