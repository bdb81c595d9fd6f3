#!/bin/bash
# One gpurun job for the round's evidence: GPU tests, smoke, bench lines of every config and the
# reference arm, launch lists (ncu per-launch durations) and one ncu --set full capture of the C3
# and C2 dominant kernels -- each ncu pass only after the plain command exited 0.
#   gpurun -- 'OUT=r02z bash tools/evidence.sh'
set -u
OUT=gpurun_out/${OUT:-evidence}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
for c in C2 C3 C1 C5 C4; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-300} --warmup 20 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_C2.json 2> $OUT/bench_ref_C2.err; echo "ref rc=$?"
timeout 900 python bench.py --sweep > $OUT/sweep.jsonl 2> $OUT/sweep.err; echo "sweep rc=$?"
for c in C3 C2; do
  python bench.py --config $c --steps 2 --warmup 1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 > $OUT/ncu_launches_$c.log 2>&1
  python tools/prof_one.py $c 3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"row_reg|st_stream" -s 2 -c 1 -o $OUT/prof_$c -f \
    python tools/prof_one.py $c 3 > $OUT/ncu_full_$c.log 2>&1
  echo "ncu $c done"
done
