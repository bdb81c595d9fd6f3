mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -x > gpurun_out/pt.log 2>&1; echo rc=$? >> gpurun_out/pt.log
timeout 120 python tools/quick_time.py C3 C3k1 C3k2 C3k8 C3r99 > gpurun_out/qt.log 2>&1
