mkdir -p gpurun_out/w10
WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w10/pytest.log
python tools/prof_run.py c3s 3 2>&1 | tail -2 | tee gpurun_out/w10/c3s.log
python tools/prof_run.py p10 3 2>&1 | tail -2 | tee -a gpurun_out/w10/c3s.log
