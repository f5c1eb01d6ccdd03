python -m pytest tests/test_cpp_api.py tests/test_acceptance.py tests/test_gpu_engine.py tests/test_gpu_store.py tests/test_gpu_cli.py -m gpu -q -rs 2>&1 | tail -30 > gpurun_out/g3_pytest.log
cat gpurun_out/g3_pytest.log
df -h /tmp | tail -1
python tools/store_bench.py --verify > gpurun_out/g3_store.json 2>&1; cat gpurun_out/g3_store.json
for c in c1 c4 c5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g3_bench_$c.json 2> gpurun_out/g3_bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/g3_bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['result_check'], d['roofline']['frac'])" || tail -5 gpurun_out/g3_bench_$c.err; done
