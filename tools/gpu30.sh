timeout 900 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/bench_c2.log | cut -c1-600
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/bench_c3.log | cut -c1-400
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench4 rc=$?"
tail -1 gpurun_out/bench_c4.log | cut -c1-400
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/bench_c1.log 2>&1; echo "bench1 rc=$?"
tail -1 gpurun_out/bench_c1.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_collect_flags|k_batch_split|k_batch_rollback' --csv --log-file gpurun_out/traffic_c2.csv python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
for k in k_batch_split k_batch_rollback k_collect_flags k_cavity_bfs k_locate; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/prof_$k python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
