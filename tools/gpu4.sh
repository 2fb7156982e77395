set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --n 1000000 --reps 3 --verbose --check > gpurun_out/probe_c2.log 2>&1; echo "probe2 rc=$?"
grep -v "^  b" gpurun_out/probe_c2.log
GDP2D_INSERT=legacy timeout 300 python tools/probe.py --n 1000000 --reps 2 > gpurun_out/probe_c2_legacy.log 2>&1; echo "probe2L rc=$?"
cat gpurun_out/probe_c2_legacy.log
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 --check > gpurun_out/probe_c3.log 2>&1; echo "probe3 rc=$?"
cat gpurun_out/probe_c3.log
