timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'], d['validation'], d['cpu_baseline']['value'])"
