mkdir -p gpurun_out/s14
timeout 900 python -m pytest tests/test_gpu_graphs.py -q -m gpu -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -3
for g in 1 0 1 0; do echo "== graphs=$g"; WHEELSIEVE_GRAPHS=$g timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['avg_launch_ms'], d['gpu_launches'], d['result_check'])"; done
WHEELSIEVE_GRAPHS=1 timeout 300 python tools/c1_overhead.py 2>&1 | tail -4
WHEELSIEVE_GRAPHS=0 timeout 300 python tools/c1_overhead.py 2>&1 | tail -4
