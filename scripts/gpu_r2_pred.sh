# predict on sweep_kernel8: GPU suite, then same-box A/B of scripts/bench_predict.py against the HEAD build
OUT=gpurun_out/pred
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $OUT/pytest_full.log; cat $OUT/pytest_full.log
for rep in 1 2 3; do
  for lab in head new; do
    if [ $lab = head ]; then L=paper_2306_14011_b200/libsurrogate_old.so; else L=paper_2306_14011_b200/libsurrogate.so; fi
    for pr in fp16 bf16; do
      SURR_LIB=$L timeout 300 python scripts/bench_predict.py --precision $pr > $OUT/pred_${lab}_${pr}_$rep.json 2>/dev/null
      python -c "
import json; d=json.loads(open('$OUT/pred_${lab}_${pr}_$rep.json').read().strip().splitlines()[-1]); print('$lab', '$pr', '%.4e'%d['value'], 'frac %.3f'%d['roofline']['frac'])"
    done
  done
done
