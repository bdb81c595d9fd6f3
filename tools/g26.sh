mkdir -p gpurun_out/r01f
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01f/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r01f/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01f/smoke.log 2>&1; echo rc=$? >> gpurun_out/r01f/smoke.log
timeout 600 python bench.py > gpurun_out/r01f/bench_C2.json 2> gpurun_out/r01f/bench_C2.err
timeout 600 python bench.py --config C3 > gpurun_out/r01f/bench_C3.json 2> gpurun_out/r01f/bench_C3.err
timeout 900 python bench.py --config C4 > gpurun_out/r01f/bench_C4.json 2> gpurun_out/r01f/bench_C4.err
timeout 900 python bench.py --config C5 > gpurun_out/r01f/bench_C5.json 2> gpurun_out/r01f/bench_C5.err
timeout 600 python bench.py --config C1 > gpurun_out/r01f/bench_C1.json 2> gpurun_out/r01f/bench_C1.err
timeout 600 python bench.py --impl reference > gpurun_out/r01f/bench_ref_C2.json 2> gpurun_out/r01f/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r01f/launches_C2.csv python bench.py --config C2 --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r01f/launches_C3.csv python bench.py --config C3 --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r01f/launches_C5.csv python bench.py --config C5 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_stream -s 3 -c 1 -o gpurun_out/r01f/prof_C2 -f python bench.py --config C2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01f/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_resident -s 3 -c 1 -o gpurun_out/r01f/prof_C3 -f python bench.py --config C3 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01f/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:st_stream -s 3 -c 1 -o gpurun_out/r01f/prof_C5 -f python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r01f/ncu_c5.log 2>&1
