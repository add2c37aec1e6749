# L2 fetch-granularity study: timings, then DRAM/L2 counters per kernel under ncu.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fetch_smi.txt 2>&1
for f in -1 0 32 64 128; do
  timeout 300 python tools/mb_fetch.py $f 1e8 >> gpurun_out/fetch_time.log 2>&1
done
for f in -1 32 64 128; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum \
    --clock-control none -k regex:mbf_ --csv --log-file gpurun_out/fetch_ncu_$f.csv python tools/mb_fetch.py $f 2e7 --once > gpurun_out/fetch_ncu_$f.log 2>&1
done
