timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
python - <<'PY'
import sys, math; sys.path.insert(0, ".")
from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host
q = QualityCriteria(math.degrees(math.asin(1/(2*math.sqrt(2)))))
pts, segs = host.generate_pslg(1_000_000, 100_000, "uniform")
m, _ = host.build_cdt(pts, segs)
with Engine(0) as e:
    e.upload(m)
    for kw in (dict(), dict(little_batch_sizing=True), dict(batch_size_cap=150000)):
        for r in range(2):
            e.reset(); rep = e.refine(q, EngineConfig(**kw))
        print(kw, f"{rep.device_seconds*1e3:.1f} ms steiner {rep.steiner_points} batches {len(rep.batches)} attempted0 {rep.batches[0].attempted}")
PY
