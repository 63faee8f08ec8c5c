OUT=gpurun_out/r2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_operands.py tests/test_gpu_parity.py tests/test_gpu_robustness.py -q -x 2>&1 | tail -15 > $OUT/pytest_k8b.log
cat $OUT/pytest_k8b.log
ab() {  # label env... -- workload
  lab=$1; wl=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $wl --no-cpu-baseline > $OUT/ab_${lab}_$wl.json 2> $OUT/ab_${lab}_$wl.err
  python - $OUT/ab_${lab}_$wl.json $lab $wl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
print(sys.argv[2], sys.argv[3], "%.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"], "alg %.0f" % r["achieved"],
      "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
}
for wl in cfg2 cfg5; do
  ab k8cb16 $wl SURR_K8CB=16
  ab k8cb0 $wl SURR_K8CB=0
  ab k3 $wl SURR_K3=1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $OUT/prof_k8_cfg2 -f python scripts/ncu_target.py cfg2 fp16 > $OUT/ncu_k8.log 2>&1
tail -3 $OUT/ncu_k8.log
