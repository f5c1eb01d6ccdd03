# L2 atomic microbench + stall-reason capture of the c3s count kernel
mkdir -p gpurun_out/s2
timeout 300 tools/_bin/mla > gpurun_out/s2/mla.txt 2>&1
cat gpurun_out/s2/mla.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_kernel -s 1 -c 1 -o gpurun_out/s2/c3s python tools/prof_run.py c3s 2 > gpurun_out/s2/ncu.log 2>&1
tail -3 gpurun_out/s2/ncu.log
