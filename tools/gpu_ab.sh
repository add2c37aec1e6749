# usage: bash tools/gpu_ab.sh "v1 v2 ..." "n dist" [ncu-kernel-regex]
mkdir -p gpurun_out
VARS=$1; WL=$2; K=${3:-}
for v in $VARS; do LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_$v.so python tools/ab_time.py $WL 5 >> gpurun_out/ab.log 2>&1; done
if [ -n "$K" ]; then
  for v in $VARS; do
    LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:$K -c 2 --csv --log-file gpurun_out/ab_ncu_$v.csv python tools/profile_step.py --n ${WL%% *} --dist ${WL##* } --steps 1 --warmup 0 > /dev/null 2>&1
  done
fi
