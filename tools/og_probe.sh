L=paper_2211_12709_b200/lib
cp $L/libdfno.so /tmp/libdfno_base.so
for v in /tmp/libdfno_base.so $L/variants/libdfno_og*.so; do
  cp $v $L/libdfno.so; touch $L/libdfno.so
  echo "=== $(basename $v)"
  for k in xmix_fwd xmix_bwd; do
    ncu --metrics launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_registers,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:xmix -c 3 python tools/time_kernel.py $k 1 2>&1 | grep -E "k_xmix|grid_size|registers|duration|dram__" | tail -7
  done
done
cp /tmp/libdfno_base.so $L/libdfno.so
