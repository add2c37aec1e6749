mkdir -p gpurun_out
python tools/dist_loopback_time.py 1e8 8 > gpurun_out/dist_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ks_|kp_" --csv --log-file gpurun_out/launches_dist.csv python tools/dist_loopback_time.py 1e8 8 > /dev/null 2>&1
