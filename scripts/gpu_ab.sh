# A/B of schedule variants (SURR_VARIANT) on one workload/precision, then a traced build's timeline
OUT=gpurun_out
WL=${1:-cfg2}; PR=${2:-fp32}; VARS=${3:-"0 1"}
for v in $VARS; do
  SURR_VARIANT=$v timeout 300 python bench.py --workload $WL --precision $PR --no-cpu-baseline > $OUT/ab_$v.json 2> $OUT/ab_$v.err
  python - $OUT/ab_$v.json $v <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print("variant", sys.argv[2], "%.4e" % d["value"], "frac %.3f issued %.3f" % (r["frac"], r["issued_frac"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print("variant", sys.argv[2], "FAILED", e)
PY
done
if [ -n "$4" ]; then
  SURR_EXTRA_FLAGS=-DSURR_TRACE python -c "from paper_2306_14011_b200.build import build_library; build_library(force=True)"
  for v in $VARS; do echo "== trace variant $v"; SURR_VARIANT=$v timeout 120 python $4; done
fi
