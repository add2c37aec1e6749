# one build->measure iteration: GPU tests (TESTS=1 all, or TESTS="-k expr"), stage times of C2/C4
# (tools/ab_time.py), optional bench lines (BENCH="c2 c4"), optional ncu launch list (NCU=c2)
mkdir -p gpurun_out
if [ "$TESTS" = 1 ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests exit $?" >> gpurun_out/t.log;
elif [ -n "$TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -x -q $TESTS > gpurun_out/t.log 2>&1; echo "tests exit $?" >> gpurun_out/t.log; fi
for cfg in ${AB:-1e8}; do timeout 600 python tools/ab_time.py $cfg uniform 5 > gpurun_out/ab_$cfg.log 2>&1; done
for c in $BENCH; do timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
if [ -n "$NCU" ]; then timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$NCU.csv python tools/ab_time.py 1e8 uniform 1 > /dev/null 2>&1; fi
