#!/bin/bash
# Round-end benches under gpurun: the driver's default command (config 3,
# K=20 W=5) and configs 1, 2, 4, 5 (device + e2e + cpu_baseline legs).
#   gpurun -- 'bash tools/gpu_benches.sh TAG'
TAG=${1:-rXX}
O=gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
echo "default rc=$?"
for c in 1 2 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/${TAG}_bench_c$c.json 2> $O/${TAG}_bench_c$c.err
  echo "c$c rc=$?"
done
for c in 3 1 2 4 5; do
  python - "$O/${TAG}_bench_c$c.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
cb = d.get("cpu_baseline") or {}
dr = d.get("e2e_dropin") or {}
print(d["config"]["workload"][:5], "dev %.2f ms" % d["ms_per_step"], "e2e %.2f ms" % (d["e2e"]["wall_s_per_step"] * 1e3),
      "dropin %.1f ms" % (dr.get("wall_s_per_step", 0) * 1e3), "steiner", d["steiner_points"], "batches", d["batches"],
      "cpu", round(cb.get("value", 0)), "frac", round(d["roofline"]["frac"], 4), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
