# quick same-box A/B against libsurrogate_old.so: parity subset (-k filter) then bench lines
# usage: bash scripts/gpu_r2_abq.sh <tag> "<workloads>" <reps> "<pytest -k filter>"
OUT=gpurun_out/$1
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "$4" 2>&1 | tail -2 > $OUT/pytest.log; cat $OUT/pytest.log
ab() {
  lab=$1; wl=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/ab_${lab}_$wl.json 2> $OUT/ab_${lab}_$wl.err
  python - $OUT/ab_${lab}_$wl.json $lab $wl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], sys.argv[3], "%.4e" % d["value"], "alg %.0f" % r["achieved"], "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
}
for rep in $(seq 1 ${3:-2}); do
  for wl in $2; do
    ab head$rep $wl SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
    ab new$rep $wl
  done
done
