for n in 50000 100000 300000; do
for dep in any mis; do
GDP2D_DEP=$dep timeout 300 python tools/probe.py --n $n --theta 30 --reps 1 2>&1 | grep "rep 0" | sed "s/^/n=$n dep=$dep /"
done
GDP2D_MODE=0 timeout 300 python tools/probe.py --n $n --theta 30 --reps 1 2>&1 | grep "rep 0" | sed "s/^/n=$n isolated /"
done
