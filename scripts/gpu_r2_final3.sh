# end-of-round evidence on the committed tree: GPU suite, smoke, bench (default, workloads,
# reference arm), launch list, ncu of the headline kernel (CSV export)
OUT=gpurun_out/final3
mkdir -p $OUT
# campaign flow check (resume across calls = same records as one call)
mkdir -p $OUT/cv
E=$((1<<36))
timeout 300 python scripts/paper_campaign.py --ckpt $OUT/cv/a.npz --end $E --chunk-log2 34 --budget-s 0.5 > $OUT/cv/a1.log 2>&1
timeout 300 python scripts/paper_campaign.py --ckpt $OUT/cv/a.npz --end $E --chunk-log2 34 --budget-s 300 > $OUT/cv/a2.log 2>&1
timeout 300 python scripts/paper_campaign.py --ckpt $OUT/cv/b.npz --end $E --chunk-log2 36 --budget-s 300 > $OUT/cv/b.log 2>&1
python - $OUT/cv <<'PY'
import json, sys
a = json.load(open(sys.argv[1] + "/a.npz.result.json")); b = json.load(open(sys.argv[1] + "/b.npz.result.json"))
print("campaign check: calls", a["calls"], "chunks-vs-one-shot identical:", a["all_idx"] == b["all_idx"] and a["all_t"] == b["all_t"],
      "oracle max rel", a["oracle_max_rel_err_at_returned"], "rate %.3e" % a["evals_per_s"])
PY
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $OUT/pytest_gpu.log; cat $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; cat $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for wl in cfg2 cfg2_fp32 cfg4 cfg3 paper cfg1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fp32-path > $OUT/launch_run.log 2>&1
rep=$OUT/prof_cfg5_fp16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $rep -f python scripts/ncu_target.py cfg5 fp16 > $OUT/ncu_cfg5.log 2>&1
ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
ncu -i $rep.ncu-rep --page source --csv --print-source sass > $rep.sass.csv 2>/dev/null
gzip -f $rep.sass.csv
for f in $OUT/bench_*.json; do python - $f <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d.get("roofline", {})
    print(sys.argv[1].split('/')[-1], "%.4e" % d["value"], "ms %.3f" % d["ms_per_step"], "frac %.3f" % r.get("frac", 0), "burst %.3f" % r.get("frac_of_burst", 0), "sust %.3f" % r.get("frac_of_sustained", 0), "e2e %.4e" % d["e2e"]["value"], d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
    if "fp32_path" in d: print("   fp32_path %.4e frac %.3f issued %.3f" % (d["fp32_path"]["value"], d["fp32_path"]["frac"], d["fp32_path"]["issued_frac"]))
    if "full_space_seconds_projected" in d.get("config", {}): print("   projected full space s", d["config"]["full_space_seconds_projected"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
