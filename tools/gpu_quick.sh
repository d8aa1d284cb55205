set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
[ -n "$NCU_KS" ] && KS="$NCU_KS" bash tools/gpu_ncu.sh > /dev/null 2>&1
tail -30 gpurun_out/pytest_gpu.log; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'])
for k,v in d['kernels'].items(): print(f'  {k:14s} {v[\"avg_ms\"]:.4f} ms x{v[\"launches_per_step\"]:.0f}  {v[\"alg_GBps\"]} GB/s')
"; tail -5 gpurun_out/bench.err
