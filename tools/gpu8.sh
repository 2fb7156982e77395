timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for mb in 2 3 4; do
  if [ $mb != 2 ]; then GDP2D_NVCC_EXTRA="-DGDP2D_SPLIT_MINB=$mb" python -c "from paper_2007_00324_b200 import build as b; b.build_cuda(force=True)"; fi
  timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2\|phase" | sed "s/^/minb=$mb c2 /"
  timeout 300 python tools/probe.py --n 5000000 --dist gaussian --reps 2 2>&1 | grep "rep 1\|phase" | sed "s/^/minb=$mb c3 /"
  GDP2D_TRACE=1 timeout 300 python tools/probe.py --n 1000000 --reps 2 > gpurun_out/trace_c2_mb$mb.log 2>&1
done
grep "^\[trace\] batch \(0\|1\|5\|10\|20\|30\|40\) " gpurun_out/trace_c2_mb2.log | tail -14
