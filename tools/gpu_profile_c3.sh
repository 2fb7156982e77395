#!/bin/bash
# North-star measurement recipe, one GPU, under gpurun:
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile_c3.sh TAG [ref]'
# Config 3 (and config 2 for the traffic table): per-batch profile, ncu launch
# list + DRAM traffic of the roofline kernels, full captures of k_batch_split /
# k_batch_rollback (a big batch and a tail batch), and with "ref" the full
# reference arm.
TAG=${1:-rXX}
O=gpurun_out
P3="tools/probe.py --n 5000000 --m 500000 --dist gaussian --reps 1"
P2="tools/probe.py --n 1000000 --m 100000 --reps 1"
timeout 600 python tools/batch_profile.py 20.704811054635428 5000000 500000 gaussian > $O/${TAG}_batch_profile_c3.txt 2>&1
echo "batch profile rc=$?"; head -7 $O/${TAG}_batch_profile_c3.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_c3.csv python $P3 > $O/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
for c in 3 2; do
  if [ $c = 3 ]; then P=$P3; else P=$P2; fi
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_collect_flags|k_collect_append|k_batch_split|k_batch_rollback' --csv \
    --log-file $O/${TAG}_traffic_c$c.csv python $P > $O/ncu_traffic.log 2>&1
  echo "ncu traffic c$c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_batch_(split|rollback)' \
  -s 2 -c 2 -o $O/${TAG}_prof_big_c3 python $P3 > $O/ncu_big.log 2>&1
echo "ncu big rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_batch_(split|rollback)' \
  -s 120 -c 2 -o $O/${TAG}_prof_tail_c3 python $P3 > $O/ncu_tail.log 2>&1
echo "ncu tail rc=$?"
if [ "$2" = "ref" ]; then
  timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $O/${TAG}_bench_reference_c3.json 2> $O/ref.err
  echo "reference rc=$?"; tail -c 600 $O/${TAG}_bench_reference_c3.json
fi
