# ncu --set full (source-level SASS with stall samples) of the ensemble pair kernel (cfg4) and kernel8 (cfg2)
OUT=gpurun_out/${1:-prof_ens}
mkdir -p $OUT
for spec in "cfg4 fp16" "cfg2 fp16"; do
  set -- $spec
  rep=$OUT/prof_$1_$2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $rep -f python scripts/ncu_target.py $1 $2 > $OUT/ncu_$1_$2.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass > $rep.sass.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source cuda > $rep.cuda.csv 2>/dev/null
  gzip -f $rep.sass.csv $rep.cuda.csv
  rm -f $rep.ncu-rep
done
ls -la $OUT
