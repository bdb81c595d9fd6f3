mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rowpipe.py -m gpu -x -q > gpurun_out/t_rp.log 2>&1; echo rc=$? >> gpurun_out/t_rp.log
timeout 300 python tools/quick_time.py C3 C3k8 C3r99 C3k2 > gpurun_out/q_rp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_pipe -s 2 -c 1 -o gpurun_out/prof_rp -f python tools/quick_time.py C3 > gpurun_out/ncu_rp.log 2>&1
