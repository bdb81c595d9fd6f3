mkdir -p gpurun_out/r01d
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01d/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r01d/pytest_gpu.log
timeout 300 python tools/quick_time.py C2 C5 C1 > gpurun_out/r01d/quick.log 2>&1
timeout 600 python bench.py --config C2 > gpurun_out/r01d/bench_C2.json 2> gpurun_out/r01d/bench_C2.err
timeout 900 python bench.py --config C5 > gpurun_out/r01d/bench_C5.json 2> gpurun_out/r01d/bench_C5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r01d/launches_C2.csv python bench.py --config C2 --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01d/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_stream -s 3 -c 1 -o gpurun_out/r01d/prof_C2 -f python bench.py --config C2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01d/ncu_f.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r01d/launches_C5.csv python bench.py --config C5 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01d/ncu_l5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_stream -s 3 -c 1 -o gpurun_out/r01d/prof_C5 -f python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01d/ncu_f5.log 2>&1
