timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -2
WHEELSIEVE_STAGE_CAP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bucket or window or c4 or c5" 2>&1 | tail -2
WHEELSIEVE_STAGE_CAP=32 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bucket or window or c4 or c5" 2>&1 | tail -2
for c in c4 c5 c4e; do bash tools/gpu/ab.sh "WHEELSIEVE_FILL_SKIP57=0" "WHEELSIEVE_FILL_SKIP57=3" $c 3; done 2>&1 | grep "==\|rep 2"
for c in c4 c5; do echo "== $c skip=1"; WHEELSIEVE_FILL_SKIP57=1 python tools/prof_run.py $c 3 | tail -1; done
