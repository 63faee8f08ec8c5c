OUT=gpurun_out/r2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py -q -x -k "ensemble or cfg4 or fused" 2>&1 | tail -15 > $OUT/pytest_ens.log
cat $OUT/pytest_ens.log
ab() {  # label wl env...
  lab=$1; wl=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $wl --no-cpu-baseline > $OUT/ab_${lab}_$wl.json 2> $OUT/ab_${lab}_$wl.err
  python - $OUT/ab_${lab}_$wl.json $lab $wl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], sys.argv[3], "%.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"], "alg %.0f" % r["achieved"],
      "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], "launch", d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
}
ab enspair cfg4 SURR_X=1
ab multipass cfg4 SURR_NO_ENS_PAIR=1
tail -5 $OUT/ab_enspair_cfg4.err
