mkdir -p gpurun_out
python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > gpurun_out/c3s_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:kd_cta_sort -s 16 -c 5 \
  -o gpurun_out/c3_small python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > gpurun_out/c3s_ncu.log 2>&1
