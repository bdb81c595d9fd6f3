mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streamthr.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_f.log 2>&1; echo rc=$? >> gpurun_out/t_f.log
timeout 300 python tools/quick_time.py C5 C2 C1 > gpurun_out/q_f.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:st_finish --csv python tools/quick_time.py C5 > gpurun_out/fin5.csv 2>&1
