set -x
timeout 120 python tools/ablate.py > gpurun_out/ablate.log 2>&1; echo "ablate rc=$?"
cut -c1-600 gpurun_out/ablate.log
timeout 300 python tools/probe.py --n 1000000 --reps 2 --verbose --check > gpurun_out/probe_c2.log 2>&1; echo "probe2 rc=$?"
grep -v "^  b" gpurun_out/probe_c2.log
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 > gpurun_out/probe_c3.log 2>&1; echo "probe3 rc=$?"
cat gpurun_out/probe_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
tail -3 gpurun_out/ncu_launch.log
for k in k_collect_flags k_cavity_bfs k_lawson_persistent k_locate k_collect_scatter k_apply_splits; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/prof_$k python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
ls -la gpurun_out
