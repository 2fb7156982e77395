#!/bin/bash
# Alternate device benches of one build under several environment settings:
#   bash tools/env_ab.sh "CFGS" ROUNDS "ENV1" "ENV2" ...   (ENV = "K=V K2=V2" or "-" for none)
CFGS=${1:-"3"}; ROUNDS=${2:-2}; shift 2
for r in $(seq $ROUNDS); do
  for c in $CFGS; do
    for e in "$@"; do
      E=""; [ "$e" != "-" ] && E="$e"
      env $E timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --dropin-steps 0 --e2e-steps 1 2>/dev/null \
        | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('r$r c$c [$e]', round(d['ms_per_step'],2), d['steiner_points'], d['batches'], 'cdt', d['validation']['cdt_violations'], 'bad', d['validation']['bad_triangles'], 'conf', d['validation']['conformity_failures'])"
    done
  done
done
