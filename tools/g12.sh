mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streamthr.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_st.log 2>&1; echo rc=$? >> gpurun_out/t_st.log
timeout 300 python tools/quick_time.py C2 C5 > gpurun_out/q_st.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:st_ --csv python tools/quick_time.py C2 > gpurun_out/st_launch.csv 2>&1
