./tools/microbench > gpurun_out/microbench.log 2>&1; cat gpurun_out/microbench.log
GDP2D_TRACE=1 timeout 300 python tools/probe.py --n 1000000 --reps 2 > gpurun_out/trace_c2.log 2>&1; echo "trace rc=$?"
grep "^\[trace\] batch \(0\|1\|5\|10\|20\|30\|40\) " gpurun_out/trace_c2.log | tail -14
