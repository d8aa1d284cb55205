# instruction count + duration of one yzt forward launch per library variant
L=paper_2211_12709_b200/lib
cp $L/libdfno.so /tmp/libdfno_base.so
for v in /tmp/libdfno_base.so $L/variants/libdfno_*.so; do
  cp $v $L/libdfno.so; touch $L/libdfno.so
  echo "=== $(basename $v)"
  python tools/time_kernel.py yzt_fwd 20
  python tools/time_kernel.py yzt_fwd_grad 20
  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum -k regex:k_yzt_fwd_tc2 -c 1 python tools/time_kernel.py yzt_fwd 1 2>&1 | grep -E "inst_executed|duration"
done 2>&1 | tee gpurun_out/inst_count.txt
cp /tmp/libdfno_base.so $L/libdfno.so
