timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bucket or window or c4 or c5" 2>&1 | tail -2
for c in c4; do
  for cap in 0 256; do echo "== $c cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py $c 3 2>&1 | tail -1; done
  echo "== $c piece 64 cap=256"; WHEELSIEVE_FILL_PIECE=64 WHEELSIEVE_STAGE_CAP=256 python tools/prof_run.py $c 3 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_run.py c4s 1 2>/dev/null | grep -v "^==" | grep fill | cut -d, -f5,15
