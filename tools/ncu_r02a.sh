set -x
bash tools/ncu_one.sh k_yzt_fwd_tc2 yzt_fwd fwd_c2
TK_GRID=33,118,64,86 bash tools/ncu_one.sh k_yzt_fwd_tc2 yzt_fwd fwd_c4
TK_GRID=33,118,64,86 bash tools/ncu_one.sh k_yzt_inv_tc3 yzt_inv inv_c4
bash tools/ncu_one.sh k_mix_bwd_tc mix_bwd mixbwd_c2
for f in gpurun_out/ncu/*.summary.txt; do echo "== $f"; cat $f; done
