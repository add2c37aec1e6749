mkdir -p gpurun_out
python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > /dev/null 2>&1
python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kc_split_level1 -s 1 -c 1 -o gpurun_out/kc_full python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/kc_full.log 2>&1
