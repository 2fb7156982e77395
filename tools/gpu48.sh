timeout 900 python -m pytest tests/test_gpu_cdt.py tests/test_gpu_refine.py -k "cdt or million or chew" -q --timeout 300 > gpurun_out/pytest_48.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_48.log; grep -E "^FAILED|Error" gpurun_out/pytest_48.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cdt.csv python tools/probe_cdt.py --n 1000000 --reps 2 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cdt_delaunay -s 1 -c 1 -o gpurun_out/prof_cdt_delaunay python tools/probe_cdt.py --n 1000000 --reps 2 > /dev/null 2>&1; echo "ncu2 rc=$?"
