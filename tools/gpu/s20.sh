timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -2
WHEELSIEVE_COOP_SKIP5=2000 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for c in c3s c2; do bash tools/gpu/ab.sh "WHEELSIEVE_COOP_SKIP5=0" "WHEELSIEVE_COOP_SKIP5=512" $c 3; done 2>&1 | grep "==\|rep 2"
for t in 128 256 1024; do echo "== c3s coop=$t"; WHEELSIEVE_COOP_SKIP5=$t python tools/prof_run.py c3s 3 | tail -1; echo "== c2 coop=$t"; WHEELSIEVE_COOP_SKIP5=$t python tools/prof_run.py c2 3 | tail -1; done
