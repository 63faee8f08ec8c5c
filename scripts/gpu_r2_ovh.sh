OUT=gpurun_out/ovh
mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29555 scripts/overhead_torchrun.py > $OUT/overhead_ws1.jsonl 2> $OUT/overhead_ws1.err
cat $OUT/overhead_ws1.jsonl; tail -3 $OUT/overhead_ws1.err
timeout 600 python bench.py --no-cpu-baseline --no-fp32-path > $OUT/bench_single.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29556 bench.py --no-cpu-baseline --no-fp32-path > $OUT/bench_torchrun1.json 2> $OUT/bench_torchrun1.err
for f in bench_single bench_torchrun1; do python -c "
import json,sys; d=json.loads(open('$OUT/$f.json').read().strip().splitlines()[-1]); print('$f', '%.4e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'e2e %.4e'%d['e2e']['value'], d['config']['parallelism'], d['gpu_launches'])"; done
