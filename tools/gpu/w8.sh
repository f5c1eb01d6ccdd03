mkdir -p gpurun_out/w8
WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w8/pytest.log
python tools/prof_run.py c3s 3 2>&1 | tail -2 | tee gpurun_out/w8/c3s.log
for cfg in p10 p11 p2e11; do
bash tools/gpu/ab.sh "WHEELSIEVE_WIDE=0" "WHEELSIEVE_WIDE=3" $cfg 3 2>&1 | grep -v "rep 0" | head -8
done | tee gpurun_out/w8/ab_sizes.log
for cfg in c2 c4 c5 c1; do python tools/prof_run.py $cfg 3 2>&1 | tail -2; done | tee gpurun_out/w8/others.log
