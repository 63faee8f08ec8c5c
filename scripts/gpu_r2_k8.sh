OUT=gpurun_out/r2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_operands.py tests/test_gpu_parity.py tests/test_gpu_robustness.py -q -x 2>&1 | tail -15 > $OUT/pytest_k8.log
cat $OUT/pytest_k8.log
SURR_LIB=build/libsurrogate_trace.so timeout 120 python scripts/trace8.py cfg2 fp16 > $OUT/trace8_cfg2.txt 2>&1
cat $OUT/trace8_cfg2.txt
for v in 0 1; do
  for wl in cfg2 cfg5; do
    SURR_K3=$v timeout 300 python bench.py --workload $wl --no-cpu-baseline > $OUT/ab8_k3${v}_$wl.json 2> $OUT/ab8_k3${v}_$wl.err
    python - $OUT/ab8_k3${v}_$wl.json $v $wl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
print("K3" if sys.argv[2] == "1" else "K8", sys.argv[3], "%.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"], "alg %.0f" % r["achieved"],
      "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
  done
done
