mkdir -p gpurun_out/w24
WHEELSIEVE_WC_SPLIT=1 WHEELSIEVE_WIDE_MIN_UNITS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w24/pytest.log
for cfg in c3s c4 c5; do
bash tools/gpu/ab.sh "WHEELSIEVE_WC_SPLIT=0" "WHEELSIEVE_WC_SPLIT=1" $cfg 3 2>&1 | grep -v "rep 0\|rep 1" | head -8
done | tee gpurun_out/w24/ab_split.log
