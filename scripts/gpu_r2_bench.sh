# bench lines of the committed tree (default + per workload)
OUT=gpurun_out/bench_$1
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for wl in cfg2 cfg2_fp32 cfg4 cfg3; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for f in $OUT/bench_*.json; do python - $f <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d.get("roofline", {})
    print(sys.argv[1].split('/')[-1], "%.4e" % d["value"], "ms %.3f" % d["ms_per_step"], "frac %.3f" % r.get("frac", 0), "burst %.3f" % r.get("frac_of_burst", 0), "sust %.3f" % r.get("frac_of_sustained", 0), "e2e %.4e" % d["e2e"]["value"], d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
    if "fp32_path" in d: print("   fp32_path %.4e frac %.3f issued %.3f" % (d["fp32_path"]["value"], d["fp32_path"]["frac"], d["fp32_path"]["issued_frac"]))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
