mkdir -p gpurun_out
python tools/dist_step.py 1e8 1 2 > gpurun_out/kp_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"kp_partition|ks_hist16" -s 2 -c 2 \
  -o gpurun_out/kp_full python tools/dist_step.py 1e8 1 2 > gpurun_out/kp_ncu.log 2>&1
