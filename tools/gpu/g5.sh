python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -3
for c in c4 c4e; do bash tools/gpu/ab.sh "WHEELSIEVE_HUGE_LOOP=1" "WHEELSIEVE_HUGE_LOOP=0" $c 3; done 2>&1 | grep "==\|rep 2"
