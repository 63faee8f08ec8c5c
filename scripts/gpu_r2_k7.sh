# kernel7 (warp-specialised) validation + same-box A/B against kernel3
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_operands.py tests/test_gpu_parity.py tests/test_gpu_robustness.py -q -x 2>&1 | tail -25 > $OUT/pytest_k7.log
cat $OUT/pytest_k7.log
for v in 0 1; do
  for wl in cfg2 cfg5; do
    SURR_K3=$v timeout 300 python bench.py --workload $wl --no-cpu-baseline > $OUT/ab_k3$v_$wl.json 2> $OUT/ab_k3${v}_$wl.err
    python - $OUT/ab_k3$v_$wl.json $v $wl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
print("K3" if sys.argv[2] == "1" else "K7", sys.argv[3], "%.4e" % d["value"], "e2e %.4e" % d["e2e"]["value"], "alg %.0f" % r["achieved"],
      "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
  done
done
SURR_NO_FUSED_MERGE=1 timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > $OUT/ab_nofuse_cfg2.json 2>&1
tail -c 600 $OUT/ab_nofuse_cfg2.json
