#!/bin/bash
# usage: tools/build_variant.sh NAME "EXTRA NVCC FLAGS" [dir-with-replacement-sources]
set -e
NAME=$1; FLAGS=$2; SRC=${3:-}
ROOT=/root/repo
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
T=/tmp/variant_$NAME; rm -rf $T; mkdir -p $T; cp -r $ROOT/paper_1909_08006_b200/csrc $T/
if [ -n "$SRC" ]; then cp $SRC/* $T/csrc/; fi
cd $T/csrc
for f in *.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I$ROOT/include -I. -I$NCCL/include -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS -c $f -o $f.o 2>/dev/null & done
for f in *.cpp; do g++ -O3 -std=c++17 -fPIC -I$ROOT/include -I. -I/usr/local/cuda/include -I$NCCL/include $(echo " $FLAGS" | grep -o " -D[^ ]*" | tr "\n" " ") -c $f -o $f.o & done
wait
mkdir -p $ROOT/vlib
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/vlib/libley_$NAME.so *.o -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo built vlib/libley_$NAME.so
