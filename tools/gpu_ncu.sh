# ncu --set full captures of the hot kernels at the C2 geometry (one GPU);
# summaries are written next to the reports, large reports are dropped.
set -x
OUT=gpurun_out/ncu
mkdir -p $OUT
KS=${KS:-"yzt_fwd yzt_fwd_grad yzt_inv xspec mix"}
for k in $KS; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:'k_(yzt|xspec|mix)' -c ${NCU_C:-2} \
    -o $OUT/$k -f python tools/kernel_driver.py $k > $OUT/$k.log 2>&1
  python tools/ncu_summary.py $OUT/$k.ncu-rep > $OUT/$k.summary.txt 2>&1
  ncu -i $OUT/$k.ncu-rep --page source --csv > $OUT/$k.source.csv 2>/dev/null
  ncu -i $OUT/$k.ncu-rep --page raw --csv > $OUT/$k.raw.csv 2>/dev/null
  gzip -f $OUT/$k.source.csv $OUT/$k.raw.csv
  [ $(stat -c %s $OUT/$k.ncu-rep) -gt 12000000 ] && rm -f $OUT/$k.ncu-rep
done
du -sh $OUT; ls -la $OUT
