# FP32-path evidence for the 3-slot 3xFP16 kernel: bench lines (cfg2, cfg5 full space, cfg1) and one ncu capture
OUT=gpurun_out/ev32
mkdir -p $OUT
timeout 600 python bench.py --workload cfg2_fp32 --no-cpu-baseline > $OUT/bench_cfg2_fp32.json 2> $OUT/bench_cfg2_fp32.err
timeout 900 python bench.py --workload cfg5 --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg5_fp32.json 2> $OUT/bench_cfg5_fp32.err
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 \
   -o $OUT/prof_cfg2_fp32 -f python scripts/ncu_target.py cfg2 fp32 > $OUT/ncu.log 2>&1
cp profiles/ncu_summary.json /tmp/ns_backup.json
python scripts/ncu_summary.py --full $OUT/prof_cfg2_fp32.ncu-rep --tag r01_fp32 > $OUT/ncu_summary.log 2>&1
cp profiles/ncu_r01_fp32.md profiles/ncu_summary.json $OUT/
rm -f $OUT/prof_cfg2_fp32.ncu-rep
cat $OUT/ncu_r01_fp32.md; for f in $OUT/bench_*.json; do echo $f; cat $f; done
