for v in base noagg base noagg; do
  LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_$v.so timeout 600 python tools/ab_opts.py 1e8 uniform $v: >> gpurun_out/abv.log 2>&1
  LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_$v.so timeout 600 python tools/ab_opts.py 2e8 skewed $v: >> gpurun_out/abv.log 2>&1
done
LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_noagg.so timeout 600 python tools/ab_opts.py 6e8 uniform noagg: >> gpurun_out/abv.log 2>&1
LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_base.so timeout 600 python tools/ab_opts.py 6e8 uniform base: >> gpurun_out/abv.log 2>&1
