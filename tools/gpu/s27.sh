timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wire.py tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -2
for i in 1 2 3; do
for c in c2 c4e; do
echo "== $c union"; python tools/prof_run.py $c 3 | tail -1
echo "== $c old"; (cd scratch/oldemit && python tools/prof_run.py $c 3 | tail -1)
done; done
for i in 1 2; do
echo "== c2 e2e union"; python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['e2e']['ms_per_step'])"
echo "== c2 e2e old"; (cd scratch/oldemit && python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['e2e']['ms_per_step'])")
done
