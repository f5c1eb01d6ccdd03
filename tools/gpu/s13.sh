# refreshed evidence after the staged fills: c4 / c4e bench lines, ncu of the staged fill kernels
mkdir -p gpurun_out/s13
for c in c4 c4e; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/s13/bench_$c.json 2> gpurun_out/s13/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/s13/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['result_check'], d['roofline']['frac'], d['clocks'])" || tail -5 gpurun_out/s13/bench_$c.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bucket_fill -s 2 -c 2 -o gpurun_out/s13/c4s_fill_staged python tools/prof_run.py c4s 2 > gpurun_out/s13/ncu.log 2>&1
tail -2 gpurun_out/s13/ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s13/c4_launches.csv python tools/prof_run.py c4 1 > gpurun_out/s13/ncu2.log 2>&1
tail -2 gpurun_out/s13/ncu2.log
