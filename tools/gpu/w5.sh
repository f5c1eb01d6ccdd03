mkdir -p gpurun_out/w5
WHEELSIEVE_SEG_WC_TRANS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w5/pytest_segtrans.log
for cfg in c2 c1 c4 c5; do
bash tools/gpu/ab.sh "WHEELSIEVE_SEG_WC_TRANS=0" "WHEELSIEVE_SEG_WC_TRANS=1" $cfg 3 2>&1 | grep -v "rep 0" 
done | tee gpurun_out/w5/ab_segtrans.log
for k in 16384 32768 49152 98304; do
echo "== skip5 $k"; WHEELSIEVE_SKIP5=$k python tools/prof_run.py c3s 3 2>&1 | tail -2
done | tee gpurun_out/w5/skip5.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/w5/bench_c3.json 2> gpurun_out/w5/bench_c3.err
python -c "import json;d=json.load(open('gpurun_out/w5/bench_c3.json'));print('c3', d['value'], d['ms_per_step'], d['e2e']['value'], d['result_check'], round(d['roofline']['frac'],4))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 1 -c 1 -o gpurun_out/w5/c3s_wide python tools/prof_run.py c3s 2 > gpurun_out/w5/ncu_c3s.log 2>&1
tail -2 gpurun_out/w5/ncu_c3s.log
