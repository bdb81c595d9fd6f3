mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C2 C5 > gpurun_out/q_ws.log 2>&1
echo "== warp sample" >> gpurun_out/q_ws.log
ATKG_ST_WARP_SAMPLE=1 timeout 300 python tools/quick_time.py C2 C5 >> gpurun_out/q_ws.log 2>&1
ATKG_ST_WARP_SAMPLE=1 timeout 900 python -m pytest tests/test_gpu_streamthr.py -m gpu -x -q > gpurun_out/t_ws.log 2>&1; echo rc=$? >> gpurun_out/t_ws.log
