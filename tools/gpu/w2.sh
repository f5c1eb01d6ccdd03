# wide kernel on by default: full GPU suite, WC-last A/B, ncu capture, c3 bench
mkdir -p gpurun_out/w2
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > gpurun_out/w2/pytest.log 2>&1
cat gpurun_out/w2/pytest.log
bash tools/gpu/ab.sh "WHEELSIEVE_WC_LAST=0" "WHEELSIEVE_WC_LAST=1" c3s 3 2>&1 | tee gpurun_out/w2/ab_wclast.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/w2/bench_c3.json 2> gpurun_out/w2/bench_c3.err
python -c "import json;d=json.load(open('gpurun_out/w2/bench_c3.json'));print('c3', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 1 -c 1 -o gpurun_out/w2/c3s_wide python tools/prof_run.py c3s 2 > gpurun_out/w2/ncu_c3s.log 2>&1
tail -3 gpurun_out/w2/ncu_c3s.log
