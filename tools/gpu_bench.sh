# tests (optional) + bench lines for the given configs
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests exit $?" >> gpurun_out/t.log; fi
for c in ${CONFIGS:-c2}; do
  extra=""; [ "$c" != c2 ] && extra="--no-e2e"
  timeout 1200 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 $extra $BENCH_EXTRA > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
done
