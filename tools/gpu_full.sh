#!/bin/bash
# One full gpurun session: GPU tests, smoke, per-config timings, bench lines, launch list
# and one ncu --set full capture of the dominant kernel per config.
#   CFGS="C2 C3" NCU_CFGS="C2" TESTS=1 bash tools/gpu_full.sh
mkdir -p gpurun_out
CFGS=${CFGS:-"C2 C3 C4 C5"}
NCU_CFGS=${NCU_CFGS:-"C2"}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
fi
if [ "${QUICK:-1}" = "1" ]; then
  timeout 600 python tools/quick_time.py ${QUICK_CFGS:-C1 C2 C3 C3k1 C3k8 C5} > gpurun_out/quick_time.log 2>&1; cat gpurun_out/quick_time.log
fi
for c in $CFGS; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?"; cat gpurun_out/bench_$c.json
done
for c in $NCU_CFGS; do
  KREGEX=${KREGEX:-}
  if [ -z "$KREGEX" ]; then
    case $c in C4) KREGEX="regex:gemm";; C3) KREGEX="regex:rowres|stage1";; *) KREGEX="regex:stage1";; esac
  fi
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_list_$c.log 2>&1
  echo "launches $c rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k "$KREGEX" -s 3 -c 1 \
      -o gpurun_out/prof_$c -f python bench.py --config $c --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_full_$c.log 2>&1
  echo "ncu full $c rc=$?"; tail -2 gpurun_out/ncu_full_$c.log
  KREGEX=""
done
