#!/bin/bash
# Quick GPU check under gpurun: a pytest selection (-k expression, or "all")
# and device-only benches of configs 3, 2 and 4 (one line each).
#   gpurun -- 'bash tools/gpu_quick.sh TAG [KEXPR]'
TAG=${1:-rXX}; K=${2:-golden}
O=gpurun_out
if [ "$K" = "all" ]; then KA=""; else KA="-k"; fi
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x $KA ${KA:+"$K"} > $O/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $O/${TAG}_pytest.log; grep -E "^FAILED|Error" $O/${TAG}_pytest.log | head -5
for c in 3 2 4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --dropin-steps 0 > $O/${TAG}_bench_c$c.json 2>$O/${TAG}_bench_c$c.err
  python -c "import json;d=json.loads(open('$O/${TAG}_bench_c$c.json').read().splitlines()[-1]);print('c$c', round(d['ms_per_step'],2), 'ms', d['steiner_points'], d['batches'], 'e2e', round(d['e2e']['wall_s_per_step']*1e3,2), 'cdt', d['validation']['cdt_violations'], 'bad', d['validation']['bad_triangles'])"
done
