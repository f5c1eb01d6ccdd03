mkdir -p gpurun_out/s5
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -2
WHEELSIEVE_STAGE_CAP=32 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bucket or window or c4 or c5" 2>&1 | tail -2
for c in c4 c5; do
  for cap in 0 128 256 512; do echo "== $c cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py $c 3 2>&1 | tail -1; done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_run.py c4s 1 2>/dev/null | grep -v "^==" | tail -12 > gpurun_out/s5/launch_c4s_256.csv
WHEELSIEVE_STAGE_CAP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_run.py c4s 1 2>/dev/null | grep -v "^==" | tail -12 > gpurun_out/s5/launch_c4s_0.csv
cat gpurun_out/s5/*.csv | cut -c1-300
