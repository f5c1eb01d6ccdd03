timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -m gpu -x 2>&1 | tail -2
for i in 1 2; do
for c in c3s c2; do
echo "== $c current"; python tools/prof_run.py $c 3 | tail -1
echo "== $c nocoop"; (cd scratch/nocoop && python tools/prof_run.py $c 3 | tail -1)
echo "== $c current SKIP5=0"; WHEELSIEVE_SKIP5=0 python tools/prof_run.py $c 3 | tail -1
done; done
