mkdir -p gpurun_out
for k in 5 10 20 100; do
  timeout 900 python bench.py --key-bytes $k --no-e2e --no-cpu --steps 5 --warmup 3 > gpurun_out/b_kb$k.json 2> gpurun_out/b_kb$k.err
done
