mkdir -p gpurun_out/w19
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > gpurun_out/w19/pytest.log 2>&1; cat gpurun_out/w19/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python - <<'PY'
import time, paper_2310_17746_b200 as ws
sv = ws.Sieve(device=0)
for i in range(6):
    t0 = time.perf_counter(); c = sv.count_range(0, 3*10**9 + 1); dt = time.perf_counter() - t0
    print("pi(3e9)", c.count, c.largest, f"{1e3*dt:.3f} ms", sv.timing().launches)
assert c.count == 144449537
PY
for c in c1 c3; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/w19/bench_$c.json 2> gpurun_out/w19/bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/w19/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4))"; done
