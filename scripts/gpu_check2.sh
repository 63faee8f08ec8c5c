# parity tests + bench lines for the precisions under development
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
for pr in fp16 fp32 fp32_3xtf32 bf16; do timeout 300 python bench.py --workload cfg2 --precision $pr --no-cpu-baseline > gpurun_out/bench_cfg2_$pr.json 2> gpurun_out/bench_cfg2_$pr.err; done
timeout 300 python bench.py --workload cfg3 --precision fp16 --no-cpu-baseline > gpurun_out/bench_cfg3_fp16.json 2> gpurun_out/bench_cfg3_fp16.err
cat gpurun_out/pytest_gpu.log; for f in gpurun_out/bench_cfg*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])" ; done
