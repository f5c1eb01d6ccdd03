# round-2 session-4 evidence: wide count kernel (3 segments per unit, one 1024-thread CTA per SM)
O=gpurun_out/f4; mkdir -p $O
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c3 c1 c2 c4 c4e c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_ncu.log 2>&1
python tools/prof_run.py c3s 2 > $O/c3s_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 1 -c 1 -o $O/c3s python tools/prof_run.py c3s 2 > $O/ncu_c3s.log 2>&1
python tools/prof_run.py c5 2 > $O/c5_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 3 -c 1 -o $O/c5 python tools/prof_run.py c5 2 > $O/ncu_c5.log 2>&1
cat $O/pytest.log $O/smoke.log
for c in c3 c1 c2 c4 c4e c5; do python -c "import json;d=json.load(open('$O/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/bench_$c.err; done
head -c 600 $O/bench_ref_c3.json
WHEELSIEVE_WIDE_MIN_UNITS=0 FUZZ_SECONDS=600 timeout 1000 python tools/fuzz_sweep.py > $O/fuzz_wide.txt 2>&1; echo "rc=$?" >> $O/fuzz_wide.txt
tail -4 $O/fuzz_wide.txt
