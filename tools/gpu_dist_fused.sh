# Fused partition + exchange checks on one GPU: dist tests, loopback timing (fused vs all-to-all), and the
# NCCL path at G=1 with the exchange phase on (C2), both transports.
mkdir -p gpurun_out
python -m pytest tests/test_dist.py -m gpu -x -q > gpurun_out/df_t.log 2>&1; echo "tests exit $?" >> gpurun_out/df_t.log
timeout 600 python tools/dist_loopback_time.py 1e8 8 > gpurun_out/df_loop.log 2>&1
for mode in "" "--alltoall"; do
  timeout 600 python bench.py --dist --exchange $mode --no-cpu --steps 5 --warmup 3 >> gpurun_out/df_bench.log 2>&1
done
timeout 600 python bench.py --dist --no-cpu --no-e2e --steps 5 --warmup 3 >> gpurun_out/df_bench.log 2>&1
