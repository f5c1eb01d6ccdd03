python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/g2_pytest.log
cat gpurun_out/g2_pytest.log
