# Round measurement: GPU tests, bench lines C1-C7 (+ C2 with 20-byte keys), ncu launch lists (C1-C4) and
# one --set full capture of the dominant kernels at C2. Everything lands in gpurun_out/ (copied to profiles/
# by hand).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi.log
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests exit $?" >> gpurun_out/t.log
for c in c2 c1 c3 c4 c5 c6 c7; do
  extra=""; [ $c != c2 ] && extra="--no-e2e"; [ $c = c5 ] || [ $c = c7 ] && extra="--steps 3"
  timeout 1200 python bench.py --config $c --warmup 3 $extra > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
done
timeout 900 python bench.py --key-bytes 20 --no-e2e --warmup 3 > gpurun_out/b_c2_kb20.json 2> gpurun_out/b_c2_kb20.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for spec in "c1 1e6 uniform 0" "c2 1e8 uniform 1" "c3 2e8 skewed 2" "c4 6e8 uniform 3"; do
  set -- $spec
  python tools/profile_step.py --n $2 --dist $3 --seed $4 --steps 1 --warmup 1 > gpurun_out/plain_$1.log 2>&1 && \
  timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$1.csv \
    python tools/profile_step.py --n $2 --dist $3 --seed $4 --steps 1 --warmup 1 > gpurun_out/ncu_$1.log 2>&1
done
python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"kd_ws_sort|ka_tile_stream" -s 2 -c 2 \
  -o gpurun_out/full_kde_c2 python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1
