# round-2 session-2 evidence after the multiple-of-5 skip and lane misses
mkdir -p gpurun_out/f3
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > gpurun_out/f3/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f3/smoke.log
for c in c3 c1 c2 c4 c4e c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/f3/bench_$c.json 2> gpurun_out/f3/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f3/bench_ref_c3.json 2> gpurun_out/f3/bench_ref_c3.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f3/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f3/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f3/launch_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_kernel -s 1 -c 1 -o gpurun_out/f3/c3s python tools/prof_run.py c3s 2 > gpurun_out/f3/ncu_c3s.log 2>&1
cat gpurun_out/f3/pytest.log gpurun_out/f3/smoke.log
for c in c3 c1 c2 c4 c4e c5; do python -c "import json;d=json.load(open('gpurun_out/f3/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/f3/bench_$c.err; done
head -c 600 gpurun_out/f3/bench_ref_c3.json
