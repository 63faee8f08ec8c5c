OUT=gpurun_out/tree
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_robustness.py -q -x -k "fused or ensemble" 2>&1 | tail -5 > $OUT/pytest_tree.log; cat $OUT/pytest_tree.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29555 scripts/overhead_torchrun.py > $OUT/overhead_ws1.jsonl 2> $OUT/overhead_ws1.err
cat $OUT/overhead_ws1.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $OUT/pytest_full.log; cat $OUT/pytest_full.log
