mkdir -p gpurun_out/w14
WHEELSIEVE_WIDE_DOUBLE=1 timeout 1500 python -m pytest tests/test_gpu_wide.py -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/w14/pytest_wide.log
WHEELSIEVE_WIDE_DOUBLE=1 WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w14/pytest_par.log
for cfg in c3s c4 c5; do
bash tools/gpu/ab.sh "WHEELSIEVE_WIDE_DOUBLE=0" "WHEELSIEVE_WIDE_DOUBLE=1" $cfg 3 2>&1 | grep -v "rep 0\|rep 1" | head -8
done | tee gpurun_out/w14/ab_double.log
for cfg in c2 c1 c4e; do python tools/prof_run.py $cfg 3 2>&1 | tail -1; done | tee gpurun_out/w14/others.log
