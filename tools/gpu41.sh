for i in 1 2; do for d in 0 1; do
GDP2D_DEVILLERS=$d timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2" | sed "s/^/dev=$d c2 /"
GDP2D_DEVILLERS=$d timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1" | sed "s/^/dev=$d c4 /"
done; done
