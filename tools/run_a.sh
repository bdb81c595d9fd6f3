set -o pipefail
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for c in C4 C2 C3 C5; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?" >> gpurun_out/bench_rc.log
done
ATKG_BENCH_SHARD=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config C5 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_C5_shard.json 2> gpurun_out/bench_C5_shard.err; echo "C5shard rc=$?" >> gpurun_out/bench_rc.log
