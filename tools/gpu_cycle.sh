# tests + A/B timing of the in-tree library (+ optional ncu --set full of one kernel at C2)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests exit $?" >> gpurun_out/t.log
for envs in ${AB_ENVS:-X=1}; do
  env $envs python tools/ab_time.py 1e8 uniform 5 1 2>&1 | sed "s/^/[$envs] /" >> gpurun_out/ab.log
  env $envs python tools/ab_time.py 2e8 skewed 5 2 2>&1 | sed "s/^/[$envs] /" >> gpurun_out/ab.log
  [ -n "$AB_C4" ] && env $envs python tools/ab_time.py 6e8 uniform 3 3 2>&1 | sed "s/^/[$envs] /" >> gpurun_out/ab.log
done
if [ -n "$NCU_K" ]; then
  python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/plain_c2.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$NCU_K -s ${NCU_S:-1} -c 1 -o gpurun_out/full_$NCU_TAG python tools/profile_step.py --n 1e8 --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1
fi
