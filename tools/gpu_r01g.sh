#!/bin/bash
# Round-1 re-entry confirmation of HEAD: GPU tests, smoke, bench lines, reference arm, C2 launch list + ncu full.
mkdir -p gpurun_out/r01g
O=gpurun_out/r01g
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in C3 C4 C5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv \
    python bench.py --config C2 --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > $O/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_stream -s 3 -c 1 \
    -o $O/prof_C2 -f python bench.py --config C2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/ncu_full.log 2>&1
echo done
