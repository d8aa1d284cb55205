# Round-2 final evidence: full GPU tests, C2 bench line (+ reference arm), C3 /
# C4-rank / C5-rank lines, launch list of the bench command, ncu summaries.
set -x
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --config C3 --no-cpu-baseline --no-e2e --no-train > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config C4rank --no-cpu-baseline --no-e2e --no-train > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config C5rank --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-train > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train > gpurun_out/b_ncu.log 2>&1
bash tools/ncu_one.sh k_yzt_fwd_tc2 yzt_fwd fwd_c2
bash tools/ncu_one.sh k_yzt_inv_tc3 yzt_inv inv_c2
bash tools/ncu_one.sh k_mix_bwd_tc mix_bwd mixbwd_c2
bash tools/ncu_one.sh k_xdft_tc xspec_fwd_ws xdft_c2
bash tools/ncu_one.sh k_xidft_tc xspec_fwd_ws xidft_c2
cat gpurun_out/pytest_gpu.log
