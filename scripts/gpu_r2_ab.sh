# GPU suite on the working tree, then same-box A/B against the HEAD build (libsurrogate_old.so)
# usage: bash scripts/gpu_r2_ab.sh <tag> "<workload> ..." [reps]
OUT=gpurun_out/$1
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $OUT/pytest_full.log; cat $OUT/pytest_full.log
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
