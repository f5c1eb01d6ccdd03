# staged fills: parity on the bucket paths, then A/B timings
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -4
WHEELSIEVE_STAGE_CAP=32 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bucket or window or c4 or c5" 2>&1 | tail -2
for c in c4 c5 c4e; do
  for cap in 0 256 512; do echo "== $c cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py $c 3 2>&1 | tail -1; done
done
for cap in 0 256; do echo "== c4 cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py c4 3 2>&1 | tail -1; done
