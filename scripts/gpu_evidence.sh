# Round evidence: full GPU suite, smoke, default bench + per-config lines, reference arm,
# ncu --set full of the bench kernels, ncu launch list of the default bench command.
set -x
OUT=gpurun_out/ev
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for wl in cfg2_fp32 cfg2_bf16 cfg3 cfg4 cfg5 cfg1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for wp in "cfg2 fp16" "cfg2 fp32" "cfg3 fp16" "cfg5 fp16"; do
  set -- $wp
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 \
     -o $OUT/prof_$1_$2 -f python scripts/ncu_target.py $1 $2 > $OUT/ncu_$1_$2.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/launch_run.log 2>&1
# summaries on the box (the .ncu-rep files are ~15 MB each; only the headline one travels back)
python scripts/ncu_summary.py --full $OUT/prof_cfg2_fp16.ncu-rep $OUT/prof_cfg2_fp32.ncu-rep $OUT/prof_cfg3_fp16.ncu-rep \
   $OUT/prof_cfg5_fp16.ncu-rep --launches $OUT/launches.csv --tag r01_final > $OUT/ncu_summary.log 2>&1
cp profiles/ncu_summary.json profiles/ncu_r01_final.md $OUT/
ncu -i $OUT/prof_cfg2_fp32.ncu-rep --page source --csv --print-source sass > $OUT/sass_cfg2_fp32.csv 2>/dev/null
rm -f $OUT/prof_cfg2_fp32.ncu-rep $OUT/prof_cfg3_fp16.ncu-rep $OUT/prof_cfg5_fp16.ncu-rep
du -sh $OUT
cat $OUT/pytest_gpu.log $OUT/smoke.log $OUT/bench_default.json
