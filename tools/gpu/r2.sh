# round-2 evidence: tests, benches per config, launch list, ncu of the headline kernel
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2/pytest.log
for c in c3 c1 c2 c4 c4e c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2/bench_ref_c3.json 2> gpurun_out/r2/bench_ref_c3.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/launch_ncu.log 2>&1
cat gpurun_out/r2/pytest.log
