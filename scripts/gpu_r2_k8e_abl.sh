# ensemble pair kernel ablations (SURR_K8E=4: no exchange, 8: nothing after a tile's last member; wrong results)
OUT=gpurun_out/${1:-k8e_abl}
mkdir -p $OUT
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
  for V in ${2:-0 4 8}; do ab v$V.$rep SURR_K8E=$V; done
done
