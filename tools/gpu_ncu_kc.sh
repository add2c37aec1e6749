mkdir -p gpurun_out
python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/kc_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kc_split_level1 -s 1 -c 1 \
  -o gpurun_out/kc_now python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/kc_ncu.log 2>&1
