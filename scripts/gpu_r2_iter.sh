# quick iteration: selected tests ($1: pytest node ids / -k expr as args) and bench lines ($2: "wl:prec ...")
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 1200 python -m pytest $1 -q -x 2>&1 | tail -25 > $OUT/pytest_iter.log
for wp in $2; do
  wl=${wp%%:*}; pr=${wp##*:}
  timeout 300 python bench.py --workload $wl --precision $pr --no-cpu-baseline > $OUT/bi_${wl}_$pr.json 2> $OUT/bi_${wl}_$pr.err
done
cat $OUT/pytest_iter.log
for wp in $2; do wl=${wp%%:*}; pr=${wp##*:}; python - $OUT/bi_${wl}_$pr.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[1], d["dtype"], "%.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"], "alg %.0f" % r["achieved"],
          "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], "launch/step %.1f" % (d["gpu_launches"] / d["steps"] / 2),
          d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
