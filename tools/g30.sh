mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C2 > gpurun_out/q_ft.log 2>&1
for th in 512 1024; do echo "== $th" >> gpurun_out/q_ft.log; ATKG_ST_FIN_THREADS=$th timeout 300 python tools/quick_time.py C2 >> gpurun_out/q_ft.log 2>&1; done
ATKG_ST_FIN_THREADS=512 timeout 900 python -m pytest tests/test_gpu_streamthr.py -m gpu -x -q > gpurun_out/t_ft.log 2>&1; echo rc=$? >> gpurun_out/t_ft.log
timeout 900 python -m pytest tests/test_gpu_streamthr.py -m gpu -x -q >> gpurun_out/t_ft.log 2>&1; echo rc=$? >> gpurun_out/t_ft.log
