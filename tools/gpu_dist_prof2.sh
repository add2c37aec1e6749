mkdir -p gpurun_out
for mode in "" "--alltoall"; do
  timeout 600 python bench.py --dist --exchange $mode --no-cpu --no-e2e --steps 5 --warmup 3 >> gpurun_out/df_bench2.log 2>&1
  timeout 600 python bench.py --config c1 --dist --exchange $mode --no-cpu --no-e2e --steps 5 --warmup 3 >> gpurun_out/df_bench2.log 2>&1
done
