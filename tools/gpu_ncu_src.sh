# source-level ncu captures: K-c at C2, the 512-tier K-d at C3 (3rd launch = level 3), kr_split at C3
mkdir -p gpurun_out
python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/src_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kc_split_level1 -s 1 -c 1 \
  -o gpurun_out/src_kc python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/src_ncu1.log 2>&1
python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > gpurun_out/src_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kd_cta_sort -s 20 -c 1 \
  -o gpurun_out/src_kd512 python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > gpurun_out/src_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kr_split -s 2 -c 1 \
  -o gpurun_out/src_kr python tools/profile_step.py --n 2e8 --dist skewed --seed 2 --steps 1 --warmup 1 > gpurun_out/src_ncu3.log 2>&1
