export GDP2D_NVCC_EXTRA="-DGDP2D_BW=1"
python -c "from paper_2007_00324_b200 import build as b; b.build_cuda(force=True)" > /dev/null 2>&1 || echo "build failed"
for cap in 1 2 3 5; do
GDP2D_EXTRAS=2 python tools/cmp_modes.py ex2 $cap 200000
GDP2D_EXTRAS=3 python tools/cmp_modes.py ex3 $cap 200000
python - <<PY
import numpy as np
a=np.load('/tmp/tris_ex2_$cap.npy'); b=np.load('/tmp/tris_ex3_$cap.npy')
sa=set(map(bytes, a)); sb=set(map(bytes, b))
print('cap $cap', len(sa), len(sb), 'only2', len(sa-sb), 'only3', len(sb-sa))
PY
done
