mkdir -p gpurun_out
python tools/mb_mem.py 1e8 l2 > gpurun_out/mb2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none -k regex:mb_ --csv --log-file gpurun_out/mb2_ncu.csv python tools/mb_mem.py 1e8 l2 > gpurun_out/mb2_ncu.log 2>&1
