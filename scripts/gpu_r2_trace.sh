OUT=gpurun_out/r2
mkdir -p gpurun_out/r2
SURR_LIB=build/libsurrogate_trace.so timeout 120 python scripts/trace7.py cfg2 fp16 > $OUT/trace7_cfg2.txt 2>&1
SURR_K3=1 SURR_LIB=build/libsurrogate_trace.so timeout 120 python scripts/trace_timeline.py cfg2 fp16 > $OUT/trace3_cfg2.txt 2>&1
timeout 120 python scripts/e2e_overhead.py > $OUT/e2e_cur.txt 2>&1
SURR_K3=1 timeout 120 python scripts/e2e_overhead.py > $OUT/e2e_cur_k3.txt 2>&1
SURR_LIB=build/libsurrogate_r1.so timeout 120 python scripts/e2e_overhead.py > $OUT/e2e_r1.txt 2>&1
cat $OUT/trace7_cfg2.txt $OUT/trace3_cfg2.txt $OUT/e2e_*.txt
