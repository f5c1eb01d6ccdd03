mkdir -p gpurun_out/w9
for m in 8 4 2 1; do
for cfg in c1 p95; do
echo "== min_units $m $cfg"; WHEELSIEVE_WIDE_MIN_UNITS=$m python tools/prof_run.py $cfg 4 2>&1 | tail -2
done; done | tee gpurun_out/w9/minunits.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 1 -c 1 -o gpurun_out/w9/c3s_wide python tools/prof_run.py c3s 2 > gpurun_out/w9/ncu_c3s.log 2>&1
tail -2 gpurun_out/w9/ncu_c3s.log
