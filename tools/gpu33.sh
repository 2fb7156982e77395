for wl in 64 256 1024 4096; do for sc in 128 256 1024; do
GDP2D_SMALL_WL=$wl GDP2D_SMALL_C=$sc timeout 300 python tools/probe.py --n 1000000 --reps 2 2>&1 | grep "rep 1" | sed "s/^/wl=$wl sc=$sc /"
done; done
