mkdir -p gpurun_out/r01c
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01c/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r01c/pytest_gpu.log
timeout 600 python bench.py --config C2 > gpurun_out/r01c/bench_C2.json 2> gpurun_out/r01c/bench_C2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r01c/launches_C2.csv python bench.py --config C2 --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01c/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_stream -s 3 -c 1 -o gpurun_out/r01c/prof_C2 -f python bench.py --config C2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01c/ncu_f.log 2>&1
