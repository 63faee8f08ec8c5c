# quick iteration: selected GPU tests (pytest -k expression in $1) + bench lines ($2: "wl:prec wl:prec ...")
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -15 > $OUT/pytest_iter.log
for wp in $2; do
  wl=${wp%%:*}; pr=${wp##*:}
  timeout 300 python bench.py --workload $wl --precision $pr --no-cpu-baseline > $OUT/bi_${wl}_$pr.json 2> $OUT/bi_${wl}_$pr.err
done
cat $OUT/pytest_iter.log
for wp in $2; do wl=${wp%%:*}; pr=${wp##*:}; python - $OUT/bi_${wl}_$pr.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[1], d["dtype"], "%.4e" % d["value"], "alg %.0f" % r["achieved"], "frac %.3f" % r["frac"],
          "issued %.3f" % r["issued_frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
