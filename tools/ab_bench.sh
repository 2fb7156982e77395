#!/bin/bash
# Alternate device benches of several engine builds on one box:
#   bash tools/ab_bench.sh "A B" "3 2" [rounds]   (abtmp/libgdp2d_<name>.so; "cur" = the tree's)
NAMES=${1:-"A B"}; CFGS=${2:-"3"}; ROUNDS=${3:-3}
for r in $(seq $ROUNDS); do
  for c in $CFGS; do
    for n in $NAMES; do
      if [ "$n" = cur ]; then L=""; else L=abtmp/libgdp2d_$n.so; fi
      GDP2D_ENGINE_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --dropin-steps 0 --e2e-steps 1 2>/dev/null \
        | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('r$r c$c $n', round(d['ms_per_step'],2), d['steiner_points'])"
    done
  done
done
