mkdir -p gpurun_out/s17
python tools/prof_run.py c2 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_kernel -s 1 -c 1 -o gpurun_out/s17/c2 python tools/prof_run.py c2 2 > gpurun_out/s17/ncu.log 2>&1
tail -2 gpurun_out/s17/ncu.log
