mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streamthr.py -m gpu -x -q > gpurun_out/t_rr.log 2>&1; echo rc=$? >> gpurun_out/t_rr.log
timeout 300 python tools/quick_time.py C3 C3r99 C3k2 C2 > gpurun_out/q_rr.log 2>&1
