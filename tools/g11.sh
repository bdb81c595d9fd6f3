mkdir -p gpurun_out/r01e
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01e/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r01e/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01e/smoke.log 2>&1; echo rc=$? >> gpurun_out/r01e/smoke.log
