python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_fullsize.py 2>&1 | tail -3
bash tools/ab_time.sh
