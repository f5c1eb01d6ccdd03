python tools/store_bench.py --L 1e15 --R 1.0001e15 --verify > gpurun_out/store_c4e.json 2>&1
python tools/store_bench.py --verify > gpurun_out/store_c2.json 2>&1
python tools/store_bench.py --text --verify > gpurun_out/store_c2_text.json 2>&1
cat gpurun_out/store_*.json
