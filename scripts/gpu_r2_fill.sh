OUT=gpurun_out/${1:-fill}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $OUT/pytest_full.log; cat $OUT/pytest_full.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29555 scripts/overhead_torchrun.py > $OUT/overhead_ws1.jsonl 2> $OUT/overhead_ws1.err
cat $OUT/overhead_ws1.jsonl
SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29556 scripts/overhead_torchrun.py > $OUT/overhead_ws1_head.jsonl 2> $OUT/overhead_ws1_head.err
echo HEAD; cat $OUT/overhead_ws1_head.jsonl
ab() {
  lab=$1; wl=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/ab_${lab}_$wl.json 2> $OUT/ab_${lab}_$wl.err
  python - $OUT/ab_${lab}_$wl.json $lab $wl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], sys.argv[3], "%.4e" % d["value"], "alg %.0f" % r["achieved"], "burst %.3f" % r["frac_of_burst"], "sust %.3f" % r["frac_of_sustained"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
}
for rep in 1 2; do
  ab head cfg2 SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
  ab new cfg2
done
ab head cfg5 SURR_LIB=paper_2306_14011_b200/libsurrogate_old.so
ab new cfg5
