mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python tools/quick_time.py C3 C3r99 C3k2 C3k8 > gpurun_out/q_sp.log 2>&1
echo "== no split" >> gpurun_out/q_sp.log
ATKG_RR_SPLIT=0 timeout 300 python tools/quick_time.py C3 C3r99 C3k2 >> gpurun_out/q_sp.log 2>&1
