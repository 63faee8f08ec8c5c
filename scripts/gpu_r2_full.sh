# full GPU suite, default bench, torchrun world-size-1 collective bench, launch list + ncu of the headline kernel
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $OUT/pytest_gpu_full.log
cat $OUT/pytest_gpu_full.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
tail -c 1500 $OUT/bench_default.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 bench.py --no-cpu-baseline > $OUT/bench_torchrun1.json 2> $OUT/bench_torchrun1.err
tail -c 600 $OUT/bench_torchrun1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $OUT/prof_k8_cfg5 -f python scripts/ncu_target.py cfg5 fp16 > $OUT/ncu_cfg5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $OUT/prof_k8_cfg2 -f python scripts/ncu_target.py cfg2 fp16 > $OUT/ncu_cfg2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $OUT/prof_k8e_cfg4 -f python scripts/ncu_target.py cfg4 fp16 > $OUT/ncu_cfg4.log 2>&1
ls -la $OUT/*.ncu-rep
