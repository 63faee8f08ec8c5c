OUT=gpurun_out/abl2
mkdir -p $OUT
for rep in 1 2; do
for v in 0 77 78; do
  for wl in cfg5 cfg2; do
    SURR_LIB=paper_2306_14011_b200/libsurrogate_abl.so SURR_VARIANT=$v timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-fp32-path > $OUT/abl_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$OUT/abl_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']; print('v$v', '$wl', '%.4e'%d['value'], 'sust %.3f'%r['frac_of_sustained'], d['clocks']['sm_mhz'])"
  done
done
done
