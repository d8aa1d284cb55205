# ncu duration / grid of the x-spectral contractions for each channel-grouping
# variant (tools/build_variant.py ogN -DDFNO_XMIX_OG=N) at C2 and at a C5 P = 8
# rank (N_x = 512, two ky per rank)
L=paper_2211_12709_b200/lib
cp $L/libdfno.so /tmp/libdfno_base.so
for v in /tmp/libdfno_base.so $L/variants/libdfno_og*.so; do
  cp $v $L/libdfno.so; touch $L/libdfno.so
  echo "=== $(basename $v)"
  for k in xmix_fwd xmix_bwd; do
    for geo in "64,64,64,32 1" "512,64,64,32 8"; do
      set -- $geo
      echo "-- $k grid $1 P $2"
      TK_GRID=$1 TK_P=$2 ncu --metrics launch__grid_size,gpu__time_duration.sum --clock-control none -k regex:xmix -c 3 \
        python tools/time_kernel.py $k 1 2>&1 | grep -E "k_xmix|grid_size|duration" | tail -3
    done
  done
done
cp /tmp/libdfno_base.so $L/libdfno.so
