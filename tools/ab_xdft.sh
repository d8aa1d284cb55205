# ncu durations of the x-DFT kernels for each variant under lib/variants at
# C2, a C5 P = 8 rank, C3 and a C4 P = 8 rank (A/B experiments)
L=paper_2211_12709_b200/lib
cp $L/libdfno.so /tmp/libdfno_base.so
for v in /tmp/libdfno_base.so $L/variants/libdfno_*.so; do
  cp $v $L/libdfno.so; touch $L/libdfno.so
  echo "=== $(basename $v)"
  for k in xdft xidft; do
    for geo in "64,64,64,32 1" "512,64,64,32 8" "128,128,128,32 1" "262,118,64,86 8"; do
      set -- $geo
      TK_GRID=$1 TK_P=$2 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_${k}_tc" -c 3 python tools/time_kernel.py $k 1 2>&1 | grep -E "duration" | tail -1 | sed "s/^/$k $1 P$2 /"
    done
  done
done
cp /tmp/libdfno_base.so $L/libdfno.so
