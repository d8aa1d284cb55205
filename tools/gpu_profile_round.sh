# Round-end evidence on one GPU: tests, bench (both arms), ncu launch list of
# the bench, ncu --set full of each hot kernel at the C2 geometry.
set -x
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
for spec in "k_yzt_fwd_tc2:yzt_fwd:yzt_fwd_act" "k_yzt_fwd_tc2:yzt_fwd_grad:yzt_fwd_grad" \
            "k_yzt_inv_tc3:yzt_inv:yzt_inv" "k_mix_bwd_tc:mix_bwd:mix_bwd" "k_mix_fwd_tma:mix_fwd:mix_fwd" \
            "k_xmix2:xspec_fwd_ws:xmix" "k_xmix_bwd2:xspec_bwd_ws:xmix_bwd" "k_xdft_s:xspec_fwd_ws:xdft" \
            "k_xidft_s:xspec_fwd_ws:xidft"; do
  IFS=: read kre tgt name <<< "$spec"
  bash tools/ncu_one.sh "$kre" "$tgt" "$name"
done
ls -la gpurun_out gpurun_out/ncu
