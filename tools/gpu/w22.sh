mkdir -p gpurun_out/w22
timeout 1500 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_virtual.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -4 | tee gpurun_out/w22/pytest.log
for cfg in c4 c5; do
for r in 5 6 8; do echo "== $cfg WIDE_PMIN=$r"; WHEELSIEVE_WIDE_PMIN=$r python tools/prof_run.py $cfg 3 2>&1 | tail -1; done
done | tee gpurun_out/w22/pmin.log
python tools/prof_run.py c4e 3 2>&1 | tail -1
