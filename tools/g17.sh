mkdir -p gpurun_out
timeout 300 python tools/cpu_cost.py > gpurun_out/cpu_cost.log 2>&1
timeout 600 python bench.py --config C2 --steps 2000 --warmup 50 --no-cpu --e2e-steps 2 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
