# swap in the diagnostics build (tools/build_variant.py prof -DDFNO_WAIT_PROF) and profile waits
L=paper_2211_12709_b200/lib
cp $L/libdfno.so /tmp/libdfno_base.so
cp $L/variants/libdfno_prof.so $L/libdfno.so; touch $L/libdfno.so
for k in ${KS:-yzt_fwd yzt_fwd_grad}; do
  python tools/wait_prof.py $k
  TK_GRID=33,118,64,86 python tools/wait_prof.py $k
done 2>&1 | tee gpurun_out/wait_prof.txt
cp /tmp/libdfno_base.so $L/libdfno.so
