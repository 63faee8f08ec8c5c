# round-2 evidence (after the top-k changes): default bench (+ fp32_path), reference arm, per-workload lines,
# launch list, ncu --set full of K1 per workload exported to CSV on the box
# (the .ncu-rep files are large: only the headline one is kept)
OUT=gpurun_out/r2q
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
tail -c 3000 $OUT/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for wl in cfg2 cfg2_fp32 cfg4 cfg3 cfg1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fp32-path > $OUT/launch_run.log 2>&1
for spec in "cfg5 fp16" "cfg2 fp16" "cfg4 fp16" "cfg5 fp32"; do
  set -- $spec
  rep=$OUT/prof_$1_$2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $rep -f python scripts/ncu_target.py $1 $2 > $OUT/ncu_$1_$2.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass > $rep.sass.csv 2>/dev/null
  gzip -f $rep.sass.csv
  [ "$1 $2" = "cfg5 fp16" ] || rm -f $rep.ncu-rep
done
ls -la $OUT
du -sh $OUT
