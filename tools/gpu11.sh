timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --n 1000000 --reps 3 --check 2>&1 | grep -v "^  b"
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_collect_flags|k_batch_split|k_batch_rollback' --csv --log-file gpurun_out/traffic_c2.csv python tools/probe.py --n 1000000 --reps 1 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c2.log | cut -c1-3000
