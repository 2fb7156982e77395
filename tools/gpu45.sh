timeout 900 python -m pytest tests/test_gpu_cdt.py -q --timeout 300 -x > gpurun_out/pytest_cdt.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_cdt.log
timeout 300 python tools/probe_cdt.py --n 1000000 --reps 3 2>&1 | tail -4
timeout 300 python tools/probe_cdt.py --n 5000000 --dist gaussian --reps 2 2>&1 | tail -3
