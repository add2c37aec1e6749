nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -o tools/libmb_mem.so tools/mb_mem.cu
