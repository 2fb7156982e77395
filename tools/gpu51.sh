for wl in 256 512 1024; do for nv in 256 1024; do
GDP2D_SMALL_WL=$wl GDP2D_SMALL_NV=$nv GDP2D_SMALL_C=$nv timeout 300 python tools/probe.py --n 1000000 --reps 3 2>&1 | grep "rep 2" | sed "s/^/c2 wl$wl nv$nv /"
GDP2D_SMALL_WL=$wl GDP2D_SMALL_NV=$nv GDP2D_SMALL_C=$nv timeout 300 python tools/probe.py --n 1000000 --theta 30 --reps 2 2>&1 | grep "rep 1" | sed "s/^/c4 wl$wl nv$nv /"
done; done
