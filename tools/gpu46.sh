timeout 900 python -m pytest tests/test_gpu_cdt.py -q --timeout 300 > gpurun_out/pytest_cdt.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/pytest_cdt.log | head -30
