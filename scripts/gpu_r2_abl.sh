# ablation of sweep_kernel8 (temporary build): which CUDA-core work bounds the tensor pipe
OUT=gpurun_out/abl
mkdir -p $OUT
for a in 0 1 8 9 2 11 4 15 31 63 32 48 0; do
  SURR_VARIANT=$((a << 16)) timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-fp32-path --steps 20 > $OUT/abl_$a.json 2> $OUT/abl_$a.err
  python - $OUT/abl_$a.json $a <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print("abl", sys.argv[2], "%.4e" % d["value"], "alg %.0f" % r["achieved"], "burst %.3f" % r["frac_of_burst"], "issued %.3f" % r["issued_frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print("abl", sys.argv[2], "FAILED", e)
PY
done
