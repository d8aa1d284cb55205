# C2 bench line + launch list (ncu, durations only) of the same command
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train > gpurun_out/b_ncu.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['step_roofline'])
for k,v in d['kernels'].items(): print(f'  {k:14s} {v[\"avg_ms\"]:.4f} ms x{v[\"launches_per_step\"]:.0f}  {v[\"alg_GBps\"]} GB/s')
"
