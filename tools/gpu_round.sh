mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests exit $?" >> gpurun_out/t.log
for c in c2 c1 c3 c4; do
  extra=""; [ $c != c2 ] && extra="--no-e2e"
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/ncu_c2.log 2>&1
