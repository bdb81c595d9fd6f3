mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C2 C5 C1 > gpurun_out/q_fl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_streamthr.py -m gpu -x -q > gpurun_out/t_fl.log 2>&1; echo rc=$? >> gpurun_out/t_fl.log
