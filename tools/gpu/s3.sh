# ncu of the two fill kernels of a c4s window and the c5 fill (data-pipe wavefronts)
mkdir -p gpurun_out/s3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bucket_fill -s 2 -c 2 -o gpurun_out/s3/c4s_fill python tools/prof_run.py c4s 2 > gpurun_out/s3/ncu.log 2>&1
tail -2 gpurun_out/s3/ncu.log
timeout 600 ncu --set full --clock-control none -k regex:bucket_fill -s 1 -c 1 -o gpurun_out/s3/c5_fill python tools/prof_run.py c5 1 > gpurun_out/s3/ncu5.log 2>&1
tail -2 gpurun_out/s3/ncu5.log
