for c in c4 c5; do
  for piece in 32 64 128; do
    for cap in 0 256; do echo "== $c piece=$piece cap=$cap"; WHEELSIEVE_FILL_PIECE=$piece WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py $c 3 2>&1 | tail -1; done
  done
done
