timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2\|phase" | sed "s/^/c2 /"
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1" | sed "s/^/c3 /"
timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1" | sed "s/^/c4 /"
done
GDP2D_TRACE=2 timeout 300 python tools/probe.py --n 1000000 --reps 1 > gpurun_out/trace2_c2.log 2>&1; python tools/trace_sum.py gpurun_out/trace2_c2.log
