#!/bin/bash
# Round-end measurement recipe (run under gpurun, one GPU):
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile.sh r01e'
# Benches of configs 1-4, the ncu launch list of config 2, DRAM traffic of the
# roofline kernels, and full captures of the top kernels, all into gpurun_out/.
TAG=${1:-rXX}
O=gpurun_out
for c in 1 2 3 4; do
  extra=""; [ $c -ge 3 ] && extra="--no-cpu-baseline"
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 $extra > $O/${TAG}_bench_c$c.log 2>&1
  echo "bench c$c rc=$?"; tail -1 $O/${TAG}_bench_c$c.log | cut -c1-200
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_c2.csv python tools/probe.py --n 1000000 --reps 1 > $O/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_collect_flags|k_batch_split|k_batch_rollback' --csv --log-file $O/${TAG}_traffic_c2.csv \
  python tools/probe.py --n 1000000 --reps 1 > $O/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
for k in k_batch_split k_batch_rollback; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o $O/${TAG}_prof_$k python tools/probe.py --n 1000000 --reps 1 > $O/ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collect_flags -s 5 -c 1 \
  -o $O/${TAG}_prof_k_collect_flags python tools/probe.py --n 1000000 --reps 1 > $O/ncu_cf.log 2>&1
echo "ncu collect rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cdt_delaunay -s 1 -c 1 \
  -o $O/${TAG}_prof_k_cdt_delaunay python tools/probe_cdt.py --n 1000000 --reps 2 > $O/ncu_cdt.log 2>&1
echo "ncu cdt rc=$?"
