# Round-2 final refresh (r02c): as gpu_round2.sh without the host-path lines (C5/C7 unchanged since r02b).
# ncu launch list of bench.py itself, DRAM launch lists for C1/C3 (profiles/ncu_traffic.json), and
# --set full captures of the dominant kernels at C4 and C2. Everything lands in gpurun_out/r2c/.
O=gpurun_out/r2c; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv > $O/smi.log
timeout 1500 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "tests exit $?" >> $O/tests.log
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1 c3 c6; do timeout 900 python bench.py --config $c --no-e2e --secondary none > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 --secondary none > $O/nb_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_bench_c4.csv python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 --secondary none > $O/nb_ncu.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for spec in "c1 1e6 uniform 0" "c2 1e8 uniform 1" "c3 2e8 skewed 2" "c4 6e8 uniform 3"; do
  set -- $spec
  timeout 1200 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$1.csv \
    python tools/profile_step.py --n $2 --dist $3 --seed $4 --steps 1 --warmup 1 > $O/ncu_$1.log 2>&1
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"kd_cta_sort" -s 6 -c 1 \
  -o $O/full_kde_c4 python tools/profile_step.py --n 6e8 --seed 3 --steps 1 --warmup 1 > $O/ncu_full_c4.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"kd_ws_sort|ka_tile_keys|kc_split_level1" -s 3 -c 3 \
  -o $O/full_c2 python tools/profile_step.py --n 1e8 --seed 1 --steps 1 --warmup 1 > $O/ncu_full_c2.log 2>&1
timeout 300 python tools/timeline.py 1e6 > $O/timeline_c1.txt 2>&1
timeout 300 python tools/timeline.py 1e6 uniform pdl=0 > $O/timeline_c1_pdl0.txt 2>&1
