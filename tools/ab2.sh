# quick check: kernel parity tests + A/B kernel timing (tools/ab_time.sh)
python -m pytest -q -x tests/test_gpu_kernels.py ${AB_TESTS} 2>&1 | tail -3
bash tools/ab_time.sh
