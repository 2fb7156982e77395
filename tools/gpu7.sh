GDP2D_TRACE=1 timeout 300 python tools/probe.py --n 1000000 --reps 2 > gpurun_out/trace_c2.log 2>&1; echo "trace rc=$?"
grep "^rep\|phase" gpurun_out/trace_c2.log
grep "^\[trace\] batch \(0\|1\|5\|10\|20\|30\|40\) " gpurun_out/trace_c2.log | tail -14
for sc in 64 128 512; do GDP2D_SMALL_C=$sc timeout 300 python tools/probe.py --n 1000000 --reps 2 2>&1 | grep "rep 1" | sed "s/^/small_c=$sc /"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
