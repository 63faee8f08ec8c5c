# FP32-path kernel (sweep_kernel6) A/B vs libsurrogate_old.so: parity subset, cfg2_fp32 lines, cfg5 fp32_path
bash scripts/gpu_r2_abq.sh ${1:-k6} "cfg2_fp32" 2 "fp32 or FP32"
OUT=gpurun_out/${1:-k6}
for lab in head new; do
  if [ $lab = head ]; then L=paper_2306_14011_b200/libsurrogate_old.so; else L=paper_2306_14011_b200/libsurrogate.so; fi
  SURR_LIB=$L timeout 600 python bench.py --no-cpu-baseline > $OUT/cfg5_$lab.json 2> $OUT/cfg5_$lab.err
  python - $OUT/cfg5_$lab.json $lab <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); f = d.get("fp32_path", {})
print(sys.argv[2], "cfg5 fp16 %.4e" % d["value"], "fp32_path", json.dumps(f)[:400])
PY
done
