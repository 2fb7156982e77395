timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
for mode in 1 2; do
GDP2D_MODE=$mode timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2\|phase" | sed "s/^/mode=$mode c2 /"
GDP2D_MODE=$mode timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase" | sed "s/^/mode=$mode c3 /"
GDP2D_MODE=$mode timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1\|phase" | sed "s/^/mode=$mode c4 /"
done
