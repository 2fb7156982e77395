timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for f in 1 0; do
GDP2D_FUSED_LAWSON=$f timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2\|phase" | sed "s/^/fused=$f c2 /"
GDP2D_FUSED_LAWSON=$f timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1" | sed "s/^/fused=$f c3 /"
GDP2D_FUSED_LAWSON=$f timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1" | sed "s/^/fused=$f c4 /"
done
GDP2D_TRACE=2 timeout 300 python tools/probe.py --n 1000000 --reps 1 > gpurun_out/trace2_c2.log 2>&1; python tools/trace_sum.py gpurun_out/trace2_c2.log
