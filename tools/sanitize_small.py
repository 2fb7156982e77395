import sys
sys.path.insert(0, '/root/repo')
from paper_2007_00324_b200 import Engine, QualityCriteria, host
pts, segs = host.generate_pslg(int(sys.argv[1]) if len(sys.argv) > 1 else 3000, (int(sys.argv[1]) if len(sys.argv) > 1 else 3000) // 10, "uniform", 5)
closed = host.close_hull(pts, segs)
with Engine(0) as eng:
    print(eng.build_cdt(pts, closed)["n_triangles"])
    rep = eng.refine(QualityCriteria(20.704811054635428))
    print(rep.steiner_points, rep.bad_triangles)
    print(eng.validate(QualityCriteria(20.704811054635428)))
