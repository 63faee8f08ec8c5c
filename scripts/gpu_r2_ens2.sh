# ensemble kernel: parity tests on the new build, then same-box A/B old vs new (cfg4)
OUT=gpurun_out/ens2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py -q -x -k "ensemble or cfg4" 2>&1 | tail -5 > $OUT/pytest.log
cat $OUT/pytest.log
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
  ab old$rep SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
  ab new$rep
done
