#!/bin/bash
# End-of-session evidence: GPU tests, smoke, bench lines (C2 default, C3, C4, C5), reference arm.
O=gpurun_out/r01z
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for c in C3 C4 C5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_C2.json 2> $O/bench_ref.err
echo done
