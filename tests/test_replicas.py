"""N>1 path of bench.py on CPU: world_size-2 gloo, the replica assignment and
the max-over-ranks aggregation (no data-path collective exists)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2007_00324_b200.replicas import Dist, assign, dist_env, replica_seed, throughput
    w, r, l = dist_env()
    d = Dist(w, r, l, backend="gloo")
    d.barrier()
    secs = 1.0 + r            # rank 1 is the slowest
    steiner = 100.0 * (r + 1)
    mx = d.max(secs)
    tot = d.sum(steiner)
    q.put((r, mx, tot, throughput(tot, mx), assign(8, w, r), replica_seed(7, r)))
    d.close()


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, mx, tot, thr, items, seed in res:
        assert mx == 2.0 and tot == 300.0 and thr == 150.0
        assert items == list(range(r, 8, 2))
        assert seed == 7 + r


def test_single_rank_is_noop():
    from paper_2007_00324_b200.replicas import Dist, assign
    d = Dist(1, 0, 0)
    d.barrier()
    assert d.max(3.0) == 3.0 and d.sum(2.0) == 2.0
    assert assign(8, 1, 0) == list(range(8))


def _refine_worker(rank, world, port, q):
    """One replica: its own PSLG (seed + rank), its own device context, a
    whole refinement, the max/sum over gloo -- bench.py's N>1 path."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    from paper_2007_00324_b200.replicas import Dist, dist_env, replica_seed, throughput
    w, r, l = dist_env()
    d = Dist(w, r, l)
    device = l % torch.cuda.device_count()   # one GPU on the test box: both replicas share it
    pts, segs = host.generate_pslg(50_000, 5_000, "uniform", replica_seed(20261017, r))
    mesh, _ = host.build_cdt(pts, segs)
    q_ = QualityCriteria(20.704811054635428)
    with Engine(device) as eng:
        eng.upload(mesh)
        d.barrier()
        rep = eng.refine(q_)
        v = eng.validate(q_)
    mx = d.max(rep.device_seconds)
    tot = d.sum(rep.steiner_points)
    q.put((r, rep.steiner_points, v["bad_triangles"], v["cdt_violations"],
           v["conformity_failures"], v["structure_failure"], mx, tot, throughput(tot, mx)))
    d.close()


@pytest.mark.gpu
def test_gloo_world2_replicas_refine(built):
    """Two ranks each refine their own mesh in their own context (same GPU on
    a one-GPU box): both results validate, they differ (distinct PSLGs), and
    the whole-job throughput is the sum over the slowest rank's time."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_refine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r, st, bad, cdt, conf, struct, mx, tot, thr in res:
        assert bad == 0 and cdt == 0 and conf == 0 and struct == 0
        assert tot == res[0][1] + res[1][1]
        assert abs(thr - tot / mx) < 1e-6 * thr
    assert res[0][1] != res[1][1]
