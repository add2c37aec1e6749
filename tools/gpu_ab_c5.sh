# A/B of library variants (vlib/) on the external path: bench.py --config c5, device clocks as recorded
mkdir -p gpurun_out
for v in $1; do
  LEY_LIBRARY_OVERRIDE=$PWD/vlib/libley_$v.so timeout 900 python bench.py --config c5 --no-cpu --steps 3 --warmup 2 \
    > gpurun_out/ab_c5_$v.json 2> gpurun_out/ab_c5_$v.err
done
