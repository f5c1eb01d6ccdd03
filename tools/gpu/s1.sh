# session-1 check of the restored checkpoint: full GPU suite, smoke, default bench
mkdir -p gpurun_out/s1
nvidia-smi -L > gpurun_out/s1/smi.txt
( time python -m pytest tests -m gpu -q 2>&1 | tail -8 ) > gpurun_out/s1/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s1/smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/s1/bench_c3.json 2> gpurun_out/s1/bench_c3.err
for c in c2 c4 c5; do python tools/prof_run.py $c 3 2>&1 | tail -2; done > gpurun_out/s1/prof.log
cat gpurun_out/s1/pytest.log gpurun_out/s1/smoke.log gpurun_out/s1/prof.log; head -c 1500 gpurun_out/s1/bench_c3.json
