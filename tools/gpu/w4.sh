mkdir -p gpurun_out/w4
WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/w4/pytest_trans.log
cat gpurun_out/w4/pytest_trans.log
WHEELSIEVE_WIDE_MIN_UNITS=0 WHEELSIEVE_WIDE_WC_LIMIT=2048 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/w4/pytest_trans2048.log
cat gpurun_out/w4/pytest_trans2048.log
bash tools/gpu/ab.sh "WHEELSIEVE_WC_TRANS=0" "WHEELSIEVE_WC_TRANS=1" c3s 3 2>&1 | tee gpurun_out/w4/ab_trans.log
for lim in 768 1536 2048 3072; do
echo "== WC limit $lim"; WHEELSIEVE_WIDE_WC_LIMIT=$lim python tools/prof_run.py c3s 3 2>&1 | tail -2
done | tee gpurun_out/w4/wclimit.log
cd tests/cpp; for i in 1 2 3; do ./_ref/cli_gpu 2>&1 | tail -1; done
