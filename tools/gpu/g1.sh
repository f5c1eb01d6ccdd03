set -x
nvidia-smi -L
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/g1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench_c3.json 2> gpurun_out/g1_bench_c3.err
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g1_bench_c2.json 2> gpurun_out/g1_bench_c2.err
tail -3 gpurun_out/g1_pytest.log; cat gpurun_out/g1_smoke.log; head -c 3000 gpurun_out/g1_bench_c3.json; tail -5 gpurun_out/g1_bench_c3.err
