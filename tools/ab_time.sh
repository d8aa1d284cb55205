# A/B kernel timing: for each variant .so under lib/variants (plus the current
# libdfno.so as "base"), swap it in and time the listed kernels at C2 and at
# one C4 rank slab.  usage: KS="yzt_fwd yzt_inv" bash tools/ab_time.sh
set -x
L=paper_2211_12709_b200/lib
cp $L/libdfno.so /tmp/libdfno_base.so
KS=${KS:-"yzt_fwd yzt_fwd_grad yzt_inv mix_fwd mix_bwd"}
for v in /tmp/libdfno_base.so $L/variants/libdfno_*.so; do
  cp $v $L/libdfno.so; touch $L/libdfno.so
  echo "=== $(basename $v)"
  for k in $KS; do python tools/time_kernel.py $k 20; done
  if [ -z "$NO_C4" ]; then for k in $KS; do TK_GRID=33,118,64,86 python tools/time_kernel.py $k 10 | sed 's/^/C4 /'; done; fi
done 2>&1 | grep -v "^+" | tee gpurun_out/ab.txt
cp /tmp/libdfno_base.so $L/libdfno.so
