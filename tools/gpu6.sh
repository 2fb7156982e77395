timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --n 1000000 --reps 3 --verbose --check > gpurun_out/probe_c2.log 2>&1; echo "probe2 rc=$?"
grep -v "^  b" gpurun_out/probe_c2.log
GDP2D_TRACE=1 timeout 300 python tools/probe.py --n 1000000 --reps 2 > gpurun_out/trace_c2.log 2>&1; echo "trace rc=$?"
grep "^\[trace\] batch \(0\|1\|5\|10\|20\|30\|40\) " gpurun_out/trace_c2.log | tail -14
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 > gpurun_out/probe_c3.log 2>&1; echo "probe3 rc=$?"
cat gpurun_out/probe_c3.log
