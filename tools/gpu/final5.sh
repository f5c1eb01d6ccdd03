# round-2 session-4 closing evidence (after the 6 S bucket threshold of wide windows)
O=gpurun_out/f5; mkdir -p $O
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c3 c4 c5 c4e c2 c1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err
done
cat $O/pytest.log $O/smoke.log
for c in c3 c1 c2 c4 c4e c5; do python -c "import json;d=json.load(open('$O/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/bench_$c.err; done
python tools/virtual_overhead.py > $O/virtual_overhead.json 2> $O/virtual_overhead.err; tail -3 $O/virtual_overhead.json
WHEELSIEVE_WIDE_MIN_UNITS=0 FUZZ_SECONDS=420 timeout 800 python tools/fuzz_sweep.py > $O/fuzz_wide.txt 2>&1; echo "rc=$?" >> $O/fuzz_wide.txt
tail -3 $O/fuzz_wide.txt
