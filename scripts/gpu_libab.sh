# A/B of two in-tree builds (libsurrogate.so vs libsurrogate_prev.so) on one workload, alternating
OUT=gpurun_out; WL=${1:-cfg2}; PR=${2:-fp16}; N=${3:-3}
for i in $(seq $N); do
  for lib in libsurrogate.so libsurrogate_prev.so; do
    SURR_LIB=paper_2306_14011_b200/$lib timeout 300 python bench.py --workload $WL --precision $PR --no-cpu-baseline > $OUT/lab.json 2> $OUT/lab.err
    python - $OUT/lab.json $lib <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], "%.4e" % d["value"], "frac %.3f" % r["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done
