# round-2 baseline: default + cfg5 bench lines, CTA-0 timeline of the headline kernel
OUT=gpurun_out/r2
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > $OUT/base_cfg2.json 2> $OUT/base_cfg2.err
timeout 300 python bench.py --workload cfg5 --no-cpu-baseline > $OUT/base_cfg5.json 2> $OUT/base_cfg5.err
SURR_LIB=build/libsurrogate_trace.so timeout 120 python scripts/trace_timeline.py cfg2 fp16 > $OUT/trace_cfg2.txt 2>&1
SURR_LIB=build/libsurrogate_trace.so timeout 120 python scripts/trace_timeline.py cfg5 fp16 > $OUT/trace_cfg5.txt 2>&1
tail -n 3 $OUT/*.json $OUT/trace_*.txt
