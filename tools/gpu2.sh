set -x
timeout 300 python tools/ablate.py > gpurun_out/ablate.log 2>&1; echo "ablate rc=$?"
cat gpurun_out/ablate.log | cut -c1-400
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench2 rc=$?"
tail -3 gpurun_out/bench_c2.log
timeout 1500 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench3 rc=$?"
tail -3 gpurun_out/bench_c3.log
