for cap in 256 128 96 64 192; do echo "== c4 cap=$cap"; WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py c4 3 | tail -1; done
for cap in 256 128 64; do echo "== c4 piece32 cap=$cap"; WHEELSIEVE_FILL_PIECE=32 WHEELSIEVE_STAGE_CAP=$cap python tools/prof_run.py c4 3 | tail -1; done
