# round 2: new GPU tests first, then the whole GPU suite, then the default bench line
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_operands.py tests/test_gpu_dist.py tests/test_gpu_robustness.py -q -x 2>&1 | tail -30 > $OUT/pytest_new.log
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -30 > $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
cat $OUT/pytest_new.log $OUT/pytest_gpu.log; tail -c 3000 $OUT/bench_default.json
