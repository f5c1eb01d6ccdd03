# wide count kernel: correctness on the goldens (forced on for every eligible launch), then A/B
mkdir -p gpurun_out/w1
for w in 3 2; do
  WHEELSIEVE_WIDE=$w WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/w1/pytest_w$w.log
  cat gpurun_out/w1/pytest_w$w.log
done
bash tools/gpu/ab.sh "WHEELSIEVE_WIDE=0" "WHEELSIEVE_WIDE=3" c3s 3 2>&1 | tee gpurun_out/w1/ab3.log
bash tools/gpu/ab.sh "WHEELSIEVE_WIDE=0" "WHEELSIEVE_WIDE=2" c3s 3 2>&1 | tee gpurun_out/w1/ab2.log
