# end-of-round check: full GPU suite, smoke, bench lines (default + every workload), reference arm
OUT=gpurun_out/final
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for wl in cfg2_fp32 cfg2_bf16 cfg3 cfg4 cfg5 paper; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
cat $OUT/pytest_gpu.log $OUT/smoke.log
for f in $OUT/bench_*.json; do python - $f <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d.get("roofline") or {}
    print(sys.argv[1].split("/")[-1], d.get("dtype"), "%.4e" % d["value"], "frac %.3f issued %.3f" % (r.get("frac", 0), r.get("issued_frac", 0)),
          (d.get("clocks") or {}).get("sm_mhz"), (d.get("e2e") or {}).get("value"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
