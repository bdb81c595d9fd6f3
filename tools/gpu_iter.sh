#!/bin/bash
# quick GPU iteration: selected GPU tests + per-config device timings
#   TESTS="tests/test_gpu_rowthr.py" QUICK="C3 C2" bash tools/gpu_iter.sh
mkdir -p gpurun_out
if [ -n "${TESTS:-}" ]; then
  timeout ${TTIME:-900} python -m pytest $TESTS -m gpu -x -q 2>&1 | tail -${TTAIL:-15} | tee gpurun_out/pytest_iter.log
fi
if [ -n "${QUICK:-}" ]; then
  timeout 600 python tools/quick_time.py $QUICK 2>&1 | tee gpurun_out/quick_iter.log
fi
if [ -n "${EXTRA:-}" ]; then bash -c "$EXTRA"; fi
