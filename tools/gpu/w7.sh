mkdir -p gpurun_out/w7
for cfg in p3e11 p5e11; do
bash tools/gpu/ab.sh "WHEELSIEVE_WIDE=0" "WHEELSIEVE_WIDE=3 WHEELSIEVE_TRANS_DEEP=0" $cfg 2 2>&1 | grep -v "rep 0" | head -4
done | tee gpurun_out/w7/ab_sizes.log
WHEELSIEVE_TRANS_DEEP=256 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 1 -c 1 -o gpurun_out/w7/c3s_deep python tools/prof_run.py c3s 2 > gpurun_out/w7/ncu_c3s.log 2>&1
tail -2 gpurun_out/w7/ncu_c3s.log
