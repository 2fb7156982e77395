for mode in 1 2 0; do
GDP2D_MODE=$mode timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2\|phase" | sed "s/^/c2 m$mode /"
GDP2D_MODE=$mode timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1" | sed "s/^/c4 m$mode /"
done
