timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for c in c3s c2 c4 c5; do bash tools/gpu/ab.sh "WHEELSIEVE_MISS_LANE=0" "WHEELSIEVE_MISS_LANE=1" $c 3; done 2>&1 | grep "==\|rep 2"
