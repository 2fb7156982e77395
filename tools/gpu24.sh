GDP2D_CHECK=1 timeout 300 python tools/probe.py --n 50000 --reps 1 2>&1 | tail -1
for n in 50000 100000 300000; do timeout 300 python tools/probe.py --n $n --theta 30 --reps 1 2>&1 | grep "rep 0" | sed "s/^/n=$n t30 /"; done
timeout 300 python tools/probe.py --n 1000000 --reps 3 --check 2>&1 | grep -v "^  b" | sed "s/^/c2 /"
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase" | sed "s/^/c3 /"
timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 --check 2>&1 | grep -v "^  b" | sed "s/^/c4 /"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
