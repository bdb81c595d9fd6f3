mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc=$? >> gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench_C2.json 2> gpurun_out/final/bench_C2.err
timeout 900 python bench.py --config C5 > gpurun_out/final/bench_C5.json 2> gpurun_out/final/bench_C5.err
timeout 600 python bench.py --config C3 > gpurun_out/final/bench_C3.json 2> gpurun_out/final/bench_C3.err
