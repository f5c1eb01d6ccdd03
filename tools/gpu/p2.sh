python tools/prof_run.py c4s 2 > gpurun_out/p2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bucket_fill -s 2 -c 2 -o gpurun_out/p2_c4s_fill python tools/prof_run.py c4s 2 > gpurun_out/p2_ncu.log 2>&1
tail -2 gpurun_out/p2_ncu.log; cat gpurun_out/p2_plain.log
