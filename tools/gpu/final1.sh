mkdir -p gpurun_out/f1
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/f1/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f1/smoke.log
cat gpurun_out/f1/pytest.log gpurun_out/f1/smoke.log
