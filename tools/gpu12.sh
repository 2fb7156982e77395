timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','e2e','roofline','gpu_launches')})"
