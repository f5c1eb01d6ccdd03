mkdir -p gpurun_out/fz3
FUZZ_SECONDS=1500 timeout 2000 python tools/fuzz_sweep.py > gpurun_out/fz3/fuzz.txt 2>&1; echo "rc=$?" >> gpurun_out/fz3/fuzz.txt
tail -4 gpurun_out/fz3/fuzz.txt
