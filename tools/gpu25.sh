GDP2D_TRACE=2 timeout 300 python tools/probe.py --n 1000000 --reps 1 > gpurun_out/trace2_c2.log 2>&1; echo "trace rc=$?"
python tools/trace_sum.py gpurun_out/trace2_c2.log
grep "counters" gpurun_out/trace2_c2.log | head -3
