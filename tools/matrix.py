"""Engine option matrix on one PSLG: every variant must validate on the device
and report its Steiner count / time.  GPU box only.
    python tools/matrix.py [n] """
import os
import subprocess
import sys

VARIANTS = [
    {},
    {"GDP2D_STANDALONE_C": "0"},
    {"GDP2D_SYNC_COLLECT": "1"},
    {"GDP2D_HALF_GRID_C": "0", "GDP2D_QUARTER_GRID_C": "0"},
    {"GDP2D_DEP": "mis"},
    {"GDP2D_MODE": "0"},
    {"GDP2D_MODE": "2"},
    {"GDP2D_HEADROOM": "1.0"},
]

CODE = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host
n = int(sys.argv[1])
pts, segs = host.generate_pslg(n, n // 10, "uniform", 5)
mesh, _ = host.build_cdt(pts, segs)
q = QualityCriteria(20.704811054635428)
with Engine(0) as eng:
    eng.upload(mesh)
    rep = eng.refine(q, EngineConfig(insert_mode=int(os.environ.get("GDP2D_MODE", "1"))))
    v = eng.validate(q)
ok = (v["structure_failure"] == 0 and v["cdt_violations"] == 0 and v["bad_triangles"] == 0
      and v["conformity_failures"] == 0 and rep.bad_triangles == 0)
print(("ok" if ok else "FAIL"), rep.steiner_points, len(rep.batches), f"{rep.device_seconds*1e3:.1f}ms",
      "" if ok else v)
'''


def main():
    n = sys.argv[1] if len(sys.argv) > 1 else "200000"
    bad = 0
    for var in VARIANTS:
        env = dict(os.environ, **var)
        r = subprocess.run([sys.executable, "-c", CODE, n], env=env, capture_output=True, text=True,
                           timeout=600)
        line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]])[-1]
        bad += not line.startswith("ok")
        print(f"{str(var):60s} {line}", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
