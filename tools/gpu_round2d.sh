# Round-2 closing measurement (r02d): bench lines at HEAD (default C4 + C2, C1, C3), the ncu launch list of
# bench.py itself, DRAM launch lists for C2/C4 (profiles/ncu_traffic.json) and a --set full capture of the
# C4 tier. Everything lands in gpurun_out/r2d/.
O=gpurun_out/r2d; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv > $O/smi.log
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1 c3; do timeout 900 python bench.py --config $c --no-e2e --secondary none > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_bench_c4.csv python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 --secondary none > $O/nb_ncu.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for spec in "c2 1e8 uniform 1" "c4 6e8 uniform 3"; do
  set -- $spec
  timeout 1200 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$1.csv \
    python tools/profile_step.py --n $2 --dist $3 --seed $4 --steps 1 --warmup 1 > $O/ncu_$1.log 2>&1
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"kd_cta_sort" -s 6 -c 1 \
  -o $O/full_kde_c4 python tools/profile_step.py --n 6e8 --seed 3 --steps 1 --warmup 1 > $O/ncu_full_c4.log 2>&1
