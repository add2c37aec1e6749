mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ascii_20gb" > gpurun_out/c67_t.log 2>&1; echo "tests exit $?" >> gpurun_out/c67_t.log
timeout 900 python bench.py --config c6 --no-e2e --steps 5 --warmup 3 > gpurun_out/b_c6.json 2> gpurun_out/b_c6.err
timeout 900 python bench.py --config c7 --steps 3 --warmup 3 > gpurun_out/b_c7.json 2> gpurun_out/b_c7.err
