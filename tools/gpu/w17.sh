mkdir -p gpurun_out/w17
WHEELSIEVE_SEG_TRANS=1 WHEELSIEVE_WIDE=0 WHEELSIEVE_WIDE_BUCKET=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/w17/pytest.log
for cfg in c2 c1 c4e; do
for t in 0 1; do echo "== $cfg SEG_TRANS=$t"; WHEELSIEVE_SEG_TRANS=$t python tools/prof_run.py $cfg 4 2>&1 | tail -2; done
done | tee gpurun_out/w17/ab.log
for m in 384 1024; do echo "== c2 SEG_TRANS=1 min $m"; WHEELSIEVE_SEG_TRANS=1 WHEELSIEVE_SEG_TRANS_MIN=$m python tools/prof_run.py c2 4 2>&1 | tail -2; done | tee -a gpurun_out/w17/ab.log
