mkdir -p gpurun_out
python tools/mb_mem.py 1e8 ${MB_CASES:-g4} > gpurun_out/mb3.log 2>&1
