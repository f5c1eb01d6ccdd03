mkdir -p gpurun_out/w21
for cfg in c4 c5; do
for r in 2 3 4 6 8 12 16; do echo "== $cfg PMIN=$r"; WHEELSIEVE_BUCKET_PMIN=$r python tools/prof_run.py $cfg 3 2>&1 | tail -1; done
done | tee gpurun_out/w21/pmin.log
