mkdir -p gpurun_out/fz2
FUZZ_SECONDS=480 timeout 900 python tools/fuzz_sweep.py > gpurun_out/fz2/fuzz.txt 2>&1; echo "rc=$?" >> gpurun_out/fz2/fuzz.txt
tail -5 gpurun_out/fz2/fuzz.txt
