python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -2
for c in c4 c5 c4e; do python tools/prof_run.py $c 4 | tail -2; done
