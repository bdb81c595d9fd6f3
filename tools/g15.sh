mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -m gpu -x -q > gpurun_out/t_s2.log 2>&1; echo rc=$? >> gpurun_out/t_s2.log
timeout 600 python bench.py --config C4 --steps 300 --warmup 10 --no-cpu --e2e-steps 2 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
ATKG_NO_RANK_SELECT=1 timeout 600 python bench.py --config C4 --steps 300 --warmup 10 --no-cpu --e2e-steps 2 > gpurun_out/b_c4_old.json 2>> gpurun_out/b_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage2 --csv python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/s2_launch.csv 2>&1
