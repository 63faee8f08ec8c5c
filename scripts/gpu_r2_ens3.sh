# unrolled-member ensemble kernel: GPU suite + same-box A/B vs HEAD (cfg4, cfg5, cfg2) + ncu of the cfg4 K1
bash scripts/gpu_r2_ab.sh ${1:-ens3} "cfg4 cfg5 cfg2" 2
OUT=gpurun_out/${1:-ens3}
rep=$OUT/prof_cfg4_fp16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $rep -f python scripts/ncu_target.py cfg4 fp16 > $OUT/ncu_cfg4.log 2>&1
ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
ncu -i $rep.ncu-rep --page source --csv --print-source sass > $rep.sass.csv 2>/dev/null
gzip -f $rep.sass.csv
rm -f $rep.ncu-rep
