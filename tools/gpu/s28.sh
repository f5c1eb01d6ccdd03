timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -2
for i in 1 2 3; do
for c in c3s c2 c4; do
echo "== $c new"; python tools/prof_run.py $c 3 | tail -1
echo "== $c base"; (cd scratch/base && python tools/prof_run.py $c 3 | tail -1)
done; done
