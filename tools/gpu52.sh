timeout 900 python -m pytest tests/test_gpu_cdt.py -q --timeout 300 > gpurun_out/pytest_cdt.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_cdt.log; grep -E "^FAILED" gpurun_out/pytest_cdt.log | head
for lv in 1 0; do
GDP2D_CDT_LEVELS=$lv timeout 300 python tools/probe_cdt.py --n 1000000 --reps 3 2>&1 | tail -1 | sed "s/^/lv$lv 1M /"
GDP2D_CDT_LEVELS=$lv timeout 300 python tools/probe_cdt.py --n 5000000 --dist gaussian --reps 2 2>&1 | tail -1 | sed "s/^/lv$lv 5M /"
done
