GDP2D_TRACE=2 timeout 300 python tools/probe.py --n 1000000 --reps 1 > gpurun_out/trace2_c2.log 2>&1; echo "trace rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
