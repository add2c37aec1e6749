# The launch list of bench.py itself (C2, kernels only: no e2e / CPU legs), after the same command ran
# clean without ncu.
mkdir -p gpurun_out
python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/nb_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_c2.csv python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 \
  > gpurun_out/nb_ncu.log 2>&1
