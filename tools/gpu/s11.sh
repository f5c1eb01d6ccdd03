timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -2
WHEELSIEVE_STAGE_CAP=32 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bucket or window or c4 or c5" 2>&1 | tail -2
for c in c4 c4e; do
  for sch in 0 1; do echo "== $c sched=$sch"; WHEELSIEVE_FILL_SCHED=$sch python tools/prof_run.py $c 3 2>&1 | tail -1; done
  for piece in 16 32; do echo "== $c sched=1 piece=$piece"; WHEELSIEVE_FILL_PIECE=$piece python tools/prof_run.py $c 3 2>&1 | tail -1; done
done
for sch in 0 1; do WHEELSIEVE_FILL_SCHED=$sch timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_run.py c4s 1 2>/dev/null | grep -v "^==" | grep -i "fill\|sieve_kernel<1" | cut -d, -f5,9,15; done
