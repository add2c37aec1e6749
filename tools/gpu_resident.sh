mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "resident or ascii_20gb or pinned or external" > gpurun_out/res_t.log 2>&1; echo "tests exit $?" >> gpurun_out/res_t.log
timeout 900 python bench.py --config c7 --steps 3 --warmup 3 > gpurun_out/b_c7.json 2> gpurun_out/b_c7.err
