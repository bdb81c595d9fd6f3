#!/bin/bash
# One gpurun session: tests, bench, launch list, full ncu capture of the stage-1 kernel.
set -o pipefail
mkdir -p gpurun_out
CFG=${CFG:-C2}
if [ "${TESTS:-1}" = "1" ]; then python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log; fi
python tools/quick_time.py C1 C2 C3 C5 2>&1 | tee gpurun_out/quick_time.log
python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; cat gpurun_out/bench_$CFG.json
if [ "${NCU:-1}" = "1" ]; then
  python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
      python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_list.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:stage1_flat -s 3 -c 1 \
      -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
