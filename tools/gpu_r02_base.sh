# Round-2 baseline evidence: GPU tests, C2 bench, C3 / C4-rank bench lines, launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --config C3 --no-cpu-baseline --no-e2e --no-train > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config C4rank --no-cpu-baseline --no-e2e --no-train > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train > gpurun_out/b_ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
