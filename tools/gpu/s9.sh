for c in c4 c4e c5; do
  for cap in 0 256; do echo "== $c cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py $c 4 2>&1 | tail -1; done
done
for c in c4 c4e; do
  for cap in 0 256; do echo "== $c cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py $c 4 2>&1 | tail -1; done
done
