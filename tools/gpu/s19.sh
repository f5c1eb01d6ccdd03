timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_graphs.py -q -m gpu -x 2>&1 | tail -2
WHEELSIEVE_SKIP5=100000000 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for c in c3s c2; do bash tools/gpu/ab.sh "WHEELSIEVE_SKIP5=0" "WHEELSIEVE_SKIP5=16384" $c 3; done 2>&1 | grep "==\|rep 2"
for t in 4096 8192 32768 65536; do echo "== c3s skip5=$t"; WHEELSIEVE_SKIP5=$t python tools/prof_run.py c3s 3 | tail -1; done
for t in 4096 8192 32768; do echo "== c2 skip5=$t"; WHEELSIEVE_SKIP5=$t python tools/prof_run.py c2 3 | tail -1; done
