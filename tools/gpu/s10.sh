timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
WHEELSIEVE_STAGE_CAP=32 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -2
