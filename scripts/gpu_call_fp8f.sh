timeout 600 python -m pytest tests/test_gpu_fp8.py -q -m gpu 2>&1 | tail -3
bash scripts/fp8_ab.sh oldq fp8f2 fp8f3 fp8f6
