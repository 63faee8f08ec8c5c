# kernel8 MODE_TOPK specialisation: GPU suite, then same-box A/B (HEAD build / any-mode / topk)
OUT=gpurun_out/k8t
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $OUT/pytest.log
cat $OUT/pytest.log
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
for rep in 1 2; do
  ab head cfg2 SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
  ab anymode cfg2 SURR_K8_ANYMODE=1
  ab topk cfg2
done
ab head cfg5 SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
ab topk cfg5
ab anymode cfg5 SURR_K8_ANYMODE=1
