mkdir -p gpurun_out
for th in 128 64 256; do
  ATKG_S2_THREADS=$th timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage2_rank --csv python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 --no-recall > gpurun_out/s2_$th.csv 2>&1
done
ATKG_S2_THREADS=256 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -m gpu -x -q -k "select or fused" > gpurun_out/t_s2.log 2>&1; echo rc=$? >> gpurun_out/t_s2.log
