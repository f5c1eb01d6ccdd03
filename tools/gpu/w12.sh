mkdir -p gpurun_out/w12
timeout 1500 python -m pytest tests/test_gpu_wide.py -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/w12/pytest_wide.log
( time python -m pytest tests -m gpu -q 2>&1 | tail -6 ) 2>&1 | tee gpurun_out/w12/pytest_all.log
python tools/prof_run.py c3s 3 2>&1 | tail -2 | tee gpurun_out/w12/c3s.log
for cfg in c4 c5; do python tools/prof_run.py $cfg 3 2>&1 | tail -2; done | tee -a gpurun_out/w12/c3s.log
