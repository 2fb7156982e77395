timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --n 1000000 --reps 3 --check 2>&1 | grep -v "^  b" | sed "s/^/c2 /"
timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase" | sed "s/^/c3 /"
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v['ms_per_launch'],4), round(v['achieved'] or 0,1), round(v['share_of_step'],3)) for k,v in d['roofline_kernels'].items()})"
