# same-box A/B of sweep_kernel8 scheduling variants (SURR_K8V), bitwise check, CTA timelines
OUT=gpurun_out/k8v
mkdir -p $OUT
for V in 0 1 2 3; do
  SURR_K8V=$V timeout 300 python - $V > $OUT/topk_$V.txt 2>&1 <<'PY'
import sys, numpy as np, torch
import paper_2306_14011_b200 as pk, workloads
wl = workloads.WORKLOADS["cfg2"]; vl = workloads.space(wl.space)
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), "fp16")
idx, t, n = h.sweep(vl, 64)
d = h.eval_range(vl, 1000000, 1000000 + 3 * 2 ** 20)
torch.cuda.synchronize()
print(" ".join(map(str, idx.cpu().numpy().tolist())))
print(" ".join("%.9g" % x for x in t.cpu().numpy().tolist()))
print("dense_sum %.10g dense_hash %d" % (float(d.double().sum()), int(np.frombuffer(d.cpu().numpy().tobytes(), np.uint32).astype(np.uint64).sum())))
PY
done
md5sum $OUT/topk_*.txt
ab() {
  lab=$1; wl=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/ab_${lab}_$wl.json 2> $OUT/ab_${lab}_$wl.err
  python - $OUT/ab_${lab}_$wl.json $lab $wl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], sys.argv[3], "%.4e" % d["value"], "alg %.0f" % r["achieved"], "burst %.3f" % r["frac_of_burst"],
          "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
}
for rep in 1 2; do
  for V in 0 1 2 3; do ab v${V}r$rep cfg2 SURR_K8V=$V; done
done
for V in 0 1 2 3; do ab v$V cfg5 SURR_K8V=$V; done
for V in 0 3; do
  SURR_LIB=paper_2306_14011_b200/libsurrogate_trace.so SURR_K8V=$V timeout 300 python scripts/trace8.py cfg2 > $OUT/trace_v$V.txt 2>&1
  cat $OUT/trace_v$V.txt
done
