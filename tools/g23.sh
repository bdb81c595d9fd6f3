mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python tools/quick_time.py C3k1 C3k2 C3r99 C3 C4x 2>/dev/null > gpurun_out/q_c3.log; timeout 300 python tools/quick_time.py C3k1 C3k2 C3r99 >> gpurun_out/q_c3.log 2>&1
