mkdir -p gpurun_out/w6
WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fuzz.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w6/pytest_deep.log
for d in 0 128 256 384 512; do
echo "== deep $d"; WHEELSIEVE_TRANS_DEEP=$d python tools/prof_run.py c3s 3 2>&1 | tail -2
done | tee gpurun_out/w6/deep.log
for cfg in p95 p10 p11; do
bash tools/gpu/ab.sh "WHEELSIEVE_WIDE=0" "WHEELSIEVE_WIDE=3" $cfg 3 2>&1 | grep -v "rep 0" | head -8
done | tee gpurun_out/w6/ab_sizes.log
