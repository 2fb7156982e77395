timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
for dep in any mis; do
GDP2D_DEP=$dep timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2\|phase" | sed "s/^/dep=$dep c2 /"
GDP2D_DEP=$dep timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase" | sed "s/^/dep=$dep c3 /"
GDP2D_DEP=$dep timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 --check 2>&1 | grep "rep 1\|phase\|check" | sed "s/^/dep=$dep c4 /"
GDP2D_DEP=$dep timeout 300 python tools/probe.py --n 100000 --m 1000 --reps 2 2>&1 | grep "rep 1" | sed "s/^/dep=$dep c1 /"
done
