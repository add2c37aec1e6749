# usage: NCU_K=regex NCU_S=skip NCU_TAG=tag [N=1e8 DIST=uniform SEED=1] bash tools/gpu_ncu1.sh
mkdir -p gpurun_out
N=${N:-1e8}; DIST=${DIST:-uniform}; SEED=${SEED:-1}
python tools/profile_step.py --n $N --dist $DIST --seed $SEED --steps 1 --warmup 1 > gpurun_out/plain_$NCU_TAG.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$NCU_K -s ${NCU_S:-0} -c 1 -o gpurun_out/full_$NCU_TAG python tools/profile_step.py --n $N --dist $DIST --seed $SEED --steps 1 --warmup 1 > gpurun_out/ncu_full_$NCU_TAG.log 2>&1
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$NCU_TAG.csv python tools/profile_step.py --n $N --dist $DIST --seed $SEED --steps 1 --warmup 1 > /dev/null 2>&1
fi
