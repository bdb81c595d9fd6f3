#!/bin/bash
# One gpurun job: GPU tests, smoke, then the bench lines named in $CONFIGS.
#   gpurun -- 'CONFIGS="C2 C3" OUT=r02a bash tools/gpu_check.sh'
set -u
OUT=gpurun_out/${OUT:-run}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
for c in ${CONFIGS:-}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-500} --warmup 20 ${BENCH_ARGS:-} > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$?"; tail -c 600 $OUT/bench_$c.json
done
