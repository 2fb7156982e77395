timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --n 1000000 --reps 3 --check --ref 2>&1 | grep -v "^  b"
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase"
timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 --check 2>&1 | grep -v "^  b"
