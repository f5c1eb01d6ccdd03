mkdir -p gpurun_out/w26
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > gpurun_out/w26/pytest.log 2>&1; cat gpurun_out/w26/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/w26/bench_c3.json 2> gpurun_out/w26/bench_c3.err
python -c "import json;d=json.load(open('gpurun_out/w26/bench_c3.json'));print('c3', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4))"
