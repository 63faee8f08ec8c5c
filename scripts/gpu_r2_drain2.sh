OUT=gpurun_out/drain2
mkdir -p $OUT
bash scripts/gpu_r2_ab.sh drain2 "cfg2 cfg5" 2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29555 scripts/overhead_torchrun.py > $OUT/overhead_ws1.jsonl 2> $OUT/overhead_ws1.err
cat $OUT/overhead_ws1.jsonl
