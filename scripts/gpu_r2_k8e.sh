# ensemble pair kernel schedule variants (SURR_K8E=V): ensemble parity tests per
# variant, then same-box A/B against the HEAD build (libsurrogate_old.so) on cfg4
OUT=gpurun_out/${1:-k8e}
mkdir -p $OUT
for V in ${2:-0 1 2 3}; do
  SURR_K8E=$V timeout 600 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py -q -x -k "ensemble or cfg4" 2>&1 | tail -2 > $OUT/pytest_v$V.log
  echo "V=$V $(tail -1 $OUT/pytest_v$V.log)"
done
ab() {
  lab=$1; shift
  env "$@" timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-fp32-path --steps 30 > $OUT/ab_$lab.json 2> $OUT/ab_$lab.err
  python - $OUT/ab_$lab.json $lab <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], "%.4e" % d["value"], "alg %.0f" % r["achieved"], "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
}
for rep in 1 2; do
  ab head$rep SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
  for V in ${2:-0 1 2 3}; do ab v$V.$rep SURR_K8E=$V; done
done
