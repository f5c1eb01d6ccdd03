# final-build profiles: launch list of the default bench, ncu of the wide kernel (c3s, one C4 window) and of C4's staged fill
O=gpurun_out/f6; mkdir -p $O
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_ncu.log 2>&1
python tools/prof_run.py c3s 2 > $O/c3s_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 1 -c 1 -o $O/c3s python tools/prof_run.py c3s 2 > $O/ncu_c3s.log 2>&1
python tools/prof_run.py c4 2 > $O/c4_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve_wide_kernel -s 5 -c 1 -o $O/c4_sieve python tools/prof_run.py c4 2 > $O/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bucket_fill_staged_kernel -s 5 -c 1 -o $O/c4_fill python tools/prof_run.py c4 2 > $O/ncu_c4f.log 2>&1
ls -la $O
