# ncu evidence for the bench's kernels: one --set full capture per workload/precision
# (second K1 launch), the launch list of the default bench command, then bench lines.
set -x
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cfg5_trained or kernel_choice or range_guard or cfg4" 2>&1 | tail -8 > $OUT/pytest_new.log
for wp in "cfg2 fp16" "cfg2 fp32" "cfg2 bf16" "cfg3 fp16"; do
  set -- $wp
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 \
     -o $OUT/prof_$1_$2 -f python scripts/ncu_target.py $1 $2 > $OUT/ncu_$1_$2.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/launch_run.log 2>&1
timeout 400 python bench.py > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 400 python bench.py --workload cfg2_fp32 --no-cpu-baseline > $OUT/bench_cfg2_fp32.json 2> $OUT/bench_cfg2_fp32.err
timeout 400 python bench.py --workload cfg3 --no-cpu-baseline > $OUT/bench_cfg3.json 2> $OUT/bench_cfg3.err
timeout 400 python bench.py --workload cfg5 --no-cpu-baseline > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
timeout 400 python bench.py --workload cfg4 --no-cpu-baseline > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
cat $OUT/pytest_new.log; ls -la $OUT
