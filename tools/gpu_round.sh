#!/bin/bash
# One GPU call: the GPU suite, the driver's default bench line, and ncu
# captures of the rollback kernel on a big (grid) and a mid-size (cluster) batch.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-rXX}; O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > $O/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $O/${TAG}_pytest.log; grep -E "^FAILED|Error" $O/${TAG}_pytest.log | head -5
timeout 900 python bench.py > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
echo "bench rc=$?"; tail -c 300 $O/${TAG}_bench_c3.json
P3="tools/probe.py --n 5000000 --m 500000 --dist gaussian --reps 1"
for s in 1 22; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_batch_rollback' \
    -s $s -c 1 -o $O/${TAG}_prof_rb${s}_c3 python $P3 > $O/ncu_rb$s.log 2>&1
  echo "ncu rb$s rc=$?"
done
