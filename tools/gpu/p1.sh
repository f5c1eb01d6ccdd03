python tools/prof_run.py c3s 2 > gpurun_out/p1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sieve_kernel -s 1 -c 1 -o gpurun_out/p1_c3s python tools/prof_run.py c3s 2 > gpurun_out/p1_ncu.log 2>&1
tail -3 gpurun_out/p1_ncu.log; cat gpurun_out/p1_plain.log
