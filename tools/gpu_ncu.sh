# ncu --set full captures of the hot kernels at the C2 geometry (one GPU).
set -x
mkdir -p gpurun_out
for k in yzt_fwd yzt_fwd_grad yzt_inv xspec mix; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:'k_(yzt|xspec|mix)' -c 3 \
    -o gpurun_out/ncu_$k -f python tools/kernel_driver.py $k > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
