# short GPU check: yzt kernel tests, C2 kernel table, C4rank kernel table
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py -k "${PYTEST_K:-yzt}" 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-e2e --no-train > /tmp/b.json
python -c "
import json; d=json.load(open('/tmp/b.json')); print('C2 value', d['value'])
for k,v in d['kernels'].items(): print('  ', k, v['avg_ms'], v['alg_GBps'])"
if [ -z "$NO_C4" ]; then
timeout 300 python bench.py --config C4rank --steps 3 --warmup 2 > /tmp/c4.json
python -c "
import json; d=json.load(open('/tmp/c4.json')); print('C4 value', d['value'])
for k,v in d['kernels'].items(): print('  ', k, v['avg_ms'], v['alg_GBps'])"
fi
