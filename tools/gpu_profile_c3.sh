#!/bin/bash
# Config-3 (north-star) measurement recipe, one GPU, under gpurun:
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile_c3.sh r02a [ref]'
# per-batch profile, ncu launch list + DRAM traffic of the roofline kernels,
# one full capture of k_batch_split, and (with "ref") the full reference arm.
TAG=${1:-rXX}
O=gpurun_out
P="tools/probe.py --n 5000000 --m 500000 --dist gaussian --reps 1"
timeout 600 python tools/batch_profile.py 20.704811054635428 5000000 500000 gaussian > $O/${TAG}_batch_profile_c3.txt 2>&1
echo "batch profile rc=$?"; head -8 $O/${TAG}_batch_profile_c3.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_c3.csv python $P > $O/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_collect_flags|k_batch_split|k_batch_rollback' --csv --log-file $O/${TAG}_traffic_c3.csv \
  python $P > $O/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_split -s 1 -c 1 \
  -o $O/${TAG}_prof_k_batch_split_c3 python $P > $O/ncu_split.log 2>&1
echo "ncu split rc=$?"
if [ "$2" = "ref" ]; then
  timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $O/${TAG}_bench_reference_c3.json 2> $O/ref.err
  echo "reference rc=$?"; tail -c 600 $O/${TAG}_bench_reference_c3.json
fi
