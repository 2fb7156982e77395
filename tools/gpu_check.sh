timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head -5
for r in 1 2; do
timeout 300 python tools/probe.py --n 100000 --m 1000 --reps 3 2>&1 | grep "rep 2" | sed "s/^/c1 /"
timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2" | sed "s/^/c2 /"
timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1" | sed "s/^/c4 /"
done
