# C2 launch list (per-stage DRAM traffic) + --set full capture of the dominant kernel (warp-specialised K-d+K-e)
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/plain_c2.log 2>&1 && \
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/ncu_c2.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:kd_ws_sort -s 1 -c 1 \
  -o gpurun_out/full_kdws_c2 python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1
