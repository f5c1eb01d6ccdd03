mkdir -p gpurun_out/w18
for cfg in c1 c2 c4e; do
for t in 0 1; do echo "== $cfg SEG_TRANS=$t min 1024"; WHEELSIEVE_SEG_TRANS=$t WHEELSIEVE_SEG_TRANS_MIN=1024 python tools/prof_run.py $cfg 5 2>&1 | tail -3; done
done | tee gpurun_out/w18/ab.log
python bench.py --config c1 --steps 50 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 bench', d['ms_per_step'], d['result_check'])"
WHEELSIEVE_SEG_TRANS=1 WHEELSIEVE_SEG_TRANS_MIN=1024 python bench.py --config c1 --steps 50 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 bench trans', d['ms_per_step'], d['result_check'])"
