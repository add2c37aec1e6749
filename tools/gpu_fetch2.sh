# TMA tensor-copy L2 promotion study (follow-up of tools/gpu_fetch.sh)
mkdir -p gpurun_out
timeout 300 python tools/mb_tma.py 1e8 > gpurun_out/tma_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum \
  --clock-control none -k regex:mbt_ --csv --log-file gpurun_out/tma_ncu.csv python tools/mb_tma.py 2e7 --once > gpurun_out/tma_ncu.log 2>&1
