mkdir -p gpurun_out/w11
python tools/prof_run.py c3s 3 2>&1 | tail -2 | tee gpurun_out/w11/c3s.log
WHEELSIEVE_WIDE_BUCKET=3 WHEELSIEVE_WIDE_MULTI=3 WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fuzz.py tests/test_gpu_virtual.py tests/test_gpu_engine.py -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/w11/pytest_b3.log
WHEELSIEVE_WIDE_BUCKET=2 WHEELSIEVE_WIDE_MULTI=2 WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/w11/pytest_b2.log
for cfg in c4 c5; do
for w in 0 2 3; do
echo "== $cfg WIDE_BUCKET=$w"; WHEELSIEVE_WIDE_BUCKET=$w python tools/prof_run.py $cfg 3 2>&1 | tail -2
done; done | tee gpurun_out/w11/ab_bucket.log
