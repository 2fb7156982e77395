#!/usr/bin/env python
"""gDP2d refinement benchmark (BASELINE.json metric: refine wall time and
Steiner points/s on one B200, against the CPU reference on the host cores).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl gdp2d|reference]

The default workload is the north-star config 3: 5M Gaussian-clustered points
+ 500K segments (SURVEY 8(d) generator, seed 20261017), radius-edge <= sqrt(2).
A *step* is one complete refinement (Algorithm 1, lines 2-9) of the workload
PSLG's initial CDT: the device-resident working mesh is restored from the
pristine copy in HBM, then refined to quality.  Line 1 (build_cdt, untimed in
the paper) runs once on the host before timing.  Under torchrun
every rank refines its own independent PSLG (seed + rank): replicas, no
data-path collective ("scaling": "weak"); the max/sum over ranks goes over gloo.

Keys beyond the base contract:
  e2e          the same metric through the C ABI context calls with HOST
               buffers: gdp2d_ctx_upload from page-locked memory (H2D), the
               refinement, gdp2d_ctx_download_to into page-locked memory (D2H),
               all inside the timed region
  e2e_dropin   the drop-in caller's path: gdp2d::refine(cdtref::Mesh&, q, cfg)
               (include/gdp2d_cdtref.hpp) on the reference's own AoS Mesh in
               pageable memory -- AoS->SoA pack, gdp2d_refine, unpack in place
  roofline     the engine kernel with the largest share of the step (CUDA events
               on the engine stream, every launch in the timed region): its
               algorithmic bytes per launch over its average
               launch time, against MEASURED_PEAKS.json hbm_gbs; traffic = ncu
               dram bytes per launch from profiles/traffic.json when present
  parity       the refined mesh against the reference's own refinement of the
               identical PSLG (tests/golden/refine_cfg.json, made by
               tests/golden/make_refine_golden.py from oracle/_ref): Steiner
               ratio, min-angle histogram total-variation distance, mean min angle
  cpu_baseline the reference (oracle/_ref, unmodified cdtref headers) on the
               IDENTICAL PSLG, host cores of this box, bounded to its first
               batches so the default run stays within minutes (the full
               reference refinement is the --impl reference arm)

--impl reference (the driver's reference arm) builds the same PSLG entirely
inside oracle/_ref (generator + close_hull + build_cdt; no product library is
loaded) and times cdtref::refine on it with all host threads.  For configs of
>= 1M points it refines ONCE, and says so.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2007_00324_b200.replicas import Dist, assign, dist_env, replica_seed  # noqa: E402

METRIC = "Refine wall-time (s) & Steiner pts/sec on 1 B200 vs CPU ref on host cores"
UNIT = "Steiner pts/s"
SEED = 20261017
B_THETA = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))
CONFIGS = {
    1: dict(n=100_000, m=1_000, dist="uniform", theta=B_THETA,
            name="cfg1: 100K uniform pts + 1K segs, radius-edge<=sqrt2"),
    2: dict(n=1_000_000, m=100_000, dist="uniform", theta=B_THETA,
            name="cfg2: 1M uniform pts + 10% segs, radius-edge<=sqrt2"),
    3: dict(n=5_000_000, m=500_000, dist="gaussian", theta=B_THETA,
            name="cfg3: 5M gaussian pts + 10% segs, radius-edge<=sqrt2"),
    4: dict(n=1_000_000, m=100_000, dist="uniform", theta=30.0,
            name="cfg4: 1M uniform pts + 10% segs, min-angle 30deg"),
    5: dict(n=2_000_000, m=200_000, dist="uniform", theta=B_THETA,
            name="cfg5: 2M uniform pts + 10% segs per GPU (replicas), radius-edge<=sqrt2"),
}
DEFAULT_CONFIG = 3
# cpu_baseline leg: the reference's first batches on the identical PSLG
# (about 15-30 s of one core at config 3); the full run is the reference arm
CPU_BASELINE_BATCHES = {1: 10000, 2: 6, 3: 1, 4: 4, 5: 4}
GOLDEN = ROOT / "tests" / "golden" / "refine_cfg.json"


def pslg_sha(pts, segs) -> str:
    """Digest of the closed PSLG (points f64 + segments u32), as in
    tests/golden/make_refine_golden.py: equal digests = identical input."""
    import numpy as np
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pts, np.float64).tobytes())
    h.update(np.ascontiguousarray(segs, np.uint32).tobytes())
    return h.hexdigest()[:32]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def loaded_repo_libs() -> list[str]:
    """In-repo shared objects mapped into this process (evidence of what ran)."""
    out = set()
    try:
        for line in open("/proc/self/maps"):
            p = line.split()[-1] if line.strip() else ""
            if p.endswith(".so") and p.startswith(str(ROOT)):
                out.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(out)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_{device}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in self.path.read_text().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows)
        load = [s for s in sm if s > 0.5 * smax] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if len(r) > 4 + k and "Active" in r[4 + k] and "Not" not in r[4 + k]})
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "samples": len(rows), "reasons": reasons}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def golden_record(config: int):
    if not GOLDEN.exists():
        return None
    return json.loads(GOLDEN.read_text()).get(f"cfg{config}")


def hist_tv(a, b) -> float:
    """Total-variation distance between two histograms (normalised)."""
    sa, sb = float(sum(a)), float(sum(b))
    if not sa or not sb:
        return 1.0
    return 0.5 * sum(abs(x / sa - y / sb) for x, y in zip(a, b))


def config_block(cfg: dict, world: int, sha: str, seed: int) -> dict:
    return {"workload": cfg["name"], "points_per_gpu": cfg["n"], "segments_per_gpu": cfg["m"],
            "distribution": cfg["dist"], "theta_deg": cfg["theta"], "seed": seed,
            "pslg_sha": sha, "parallelism": f"replicas{world}" if world > 1 else "single",
            "l2": "512 MB flush before every step; mesh > L2"}


# ---------------------------------------------------------------------------------------
# reference arm: the unmodified cdtref headers (oracle/_ref) only
# ---------------------------------------------------------------------------------------

def run_reference_arm(a, world, rank):
    if rank != 0:
        return 0
    from oracle.ref import ref_workload
    from paper_2007_00324_b200.gdp2d import QualityCriteria   # pure Python (no library)
    cfg = CONFIGS[a.config]
    seed = replica_seed(SEED, 0)
    t0 = time.perf_counter()
    pts, closed, base = ref_workload(cfg["n"], cfg["m"], cfg["dist"], seed)
    setup_s = time.perf_counter() - t0
    sha = pslg_sha(pts, closed)
    q = QualityCriteria(cfg["theta"])
    cores = os.cpu_count() or 1
    big = cfg["n"] >= 1_000_000
    runs = 1 if big else max(1, a.steps)
    warm = 0 if big else max(0, a.warmup)
    for _ in range(warm):
        base.clone().refine(q, executors=cores)
    st, secs, batches = [], [], []
    for _ in range(runs):
        m = base.clone()
        rep = m.refine(q, executors=cores)
        st.append(rep.steiner_points)
        secs.append(rep.wall_seconds)
        batches.append(len(rep.batches))
    total = sum(secs)
    value = sum(st) / total
    sample = (f"cdtref::refine (oracle/_ref: the unmodified reference headers, g++ -O3) on the "
              f"identical {cfg['name'].split(':')[0]} PSLG (pslg_sha {sha}), "
              f"ExecutionMode::Parallel with {cores} executors, {runs} full run(s)"
              + (" -- one run for configs >= 1M points (BASELINE.md section 2), "
                 f"{a.steps} requested" if big else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": runs, "requested_steps": a.steps, "warmup": warm, "requested_warmup": a.warmup,
        "ms_per_step": total / runs * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, world, sha, seed),
        "same_config": True,
        "refine_wall_s": total / runs, "steiner_points": st[-1], "batches": batches[-1],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup_s,
        "native_so_loaded": loaded_repo_libs(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------

LINE1 = {}   # first workload's PSLG + reference build_cdt time


def make_workload(cfg: dict, seed: int):
    from paper_2007_00324_b200 import host
    pts, segs = host.generate_pslg(cfg["n"], cfg["m"], cfg["dist"], seed)
    t0 = time.perf_counter()
    mesh, closed = host.build_cdt(pts, segs)
    if not LINE1:
        LINE1.update(pts=pts, closed=closed, ref_s=time.perf_counter() - t0,
                     ref_tris=int(mesh.tri_alive.sum()))
    return mesh, pslg_sha(pts, closed)


def line1_device(device: int) -> dict:
    """Line 1 (build_cdt, cdt.hpp:483) on the device for the same PSLG: median
    of 3 builds after one warm-up, beside the reference's host build time
    measured while preparing the workload (not part of the refine metric)."""
    from paper_2007_00324_b200 import Engine
    with Engine(device) as e:
        e.build_cdt(LINE1["pts"], LINE1["closed"])
        runs = [e.build_cdt(LINE1["pts"], LINE1["closed"]) for _ in range(3)]
    ms = sorted(r["seconds"] * 1e3 for r in runs)[1]
    r = runs[-1]
    return {"device_ms": ms, "reference_host_s": LINE1["ref_s"],
            "speedup": LINE1["ref_s"] * 1e3 / ms, "triangles": r["n_triangles"],
            "same_triangle_count": r["n_triangles"] == LINE1["ref_tris"],
            "insert_rounds": r["insert_rounds"], "recover_rounds": r["recover_rounds"],
            "note": "device build of the bench PSLG (untimed in the paper); "
                    "triangle-set parity: tests/test_gpu_cdt.py"}


def mesh_bytes(m) -> int:
    return sum(getattr(m, k).nbytes for k in ("xy", "vert_kind", "vert_birth", "vert_alive",
                                              "vert_tri", "tri_v", "tri_n", "tri_seg", "tri_alive",
                                              "seg_v", "seg_parent", "seg_encroached", "seg_alive",
                                              "seg_tri"))


def cpu_baseline_leg(cfg: dict, config: int, mesh, sha: str) -> dict:
    """The reference (oracle/_ref) on the identical initial CDT, bounded to its
    first CPU_BASELINE_BATCHES batches, one core (EngineConfig{} is sequential)."""
    from oracle.ref import RefMesh
    from paper_2007_00324_b200 import EngineConfig, QualityCriteria
    cap = CPU_BASELINE_BATCHES[config]
    rm = RefMesh.from_mesh(mesh)
    rep = rm.refine(QualityCriteria(cfg["theta"]), EngineConfig(iteration_cap=cap))
    full = not rep.iteration_cap_hit
    return {"value": rep.steiner_points / rep.wall_seconds, "unit": UNIT, "cores": 1,
            "kind": "reference", "cpu_model": cpu_model(),
            "sample": (f"cdtref::refine (oracle/_ref, g++ -O3, EngineConfig{{}} sequential) on the "
                       f"identical PSLG (pslg_sha {sha}), "
                       + ("the full refinement" if full else
                          f"its first {len(rep.batches)} batches (iteration_cap={cap}); "
                          "the tail batches are slower per point, so this overstates the "
                          "reference's full-run rate. The full run is --impl reference")),
            "seconds": rep.wall_seconds, "steiner": rep.steiner_points,
            "batches": len(rep.batches)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="gdp2d", choices=["gdp2d", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps")
    ap.add_argument("--dropin-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    world, rank, local = dist_env()
    if a.impl == "reference":
        return run_reference_arm(a, world, rank)

    import torch

    from paper_2007_00324_b200 import Engine, QualityCriteria
    from paper_2007_00324_b200 import _abi as A
    from paper_2007_00324_b200 import host

    dist = Dist(world, rank, local)
    device = local % max(1, torch.cuda.device_count())   # ranks share a GPU only on a smaller box
    torch.cuda.set_device(device)
    cfg = CONFIGS[a.config]
    q = QualityCriteria(cfg["theta"])
    # config 5: a batch of 8 independent PSLGs spread round-robin over the
    # ranks; otherwise one PSLG per rank (weak scaling)
    items = assign(8, world, rank) if a.config == 5 else [0]
    seeds = [replica_seed(SEED, rank if a.config != 5 else 0, it) for it in items]
    t0 = time.time()
    work = [make_workload(cfg, s) for s in seeds]
    meshes = [w[0] for w in work]
    sha = work[0][1]
    setup_s = time.time() - t0
    lib = A.engine()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")  # > 126 MB L2

    engines = []
    for mm in meshes:
        e = Engine(device)
        e.upload(mm)
        engines.append(e)
    for _ in range(max(a.warmup, 0)):
        for e in engines:
            e.reset()
            e.refine(q)

    # ---- timed region: K device-resident steps ----
    reps = []
    step_ms = []
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.gdp2d_kernel_launches()
    with ClockSampler(device) as clk:
        host_t0 = time.perf_counter()
        for _ in range(a.steps):
            ms = 0.0
            for e in engines:
                flush.zero_()                       # evict L2 before every refine
                torch.cuda.synchronize()
                e.reset()
                rep = e.refine(q)
                reps.append(rep)
                ms += rep.device_seconds * 1e3
            step_ms.append(ms)
        torch.cuda.synchronize()
        host_s = time.perf_counter() - host_t0
    launches = lib.gdp2d_kernel_launches() - launches0
    dist.barrier()
    dev_s = sum(step_ms) / 1e3
    dev_s_max = dist.max(dev_s)
    steiner_local = sum(r.steiner_points for r in reps)
    steiner_all = dist.sum(steiner_local)
    value = steiner_all / dev_s_max
    last = reps[-1]

    # ---- e2e: the C ABI context calls with HOST buffers (page-locked) ----
    # Every step: H2D of the input mesh from pinned host memory (Engine.upload
    # -> gdp2d_ctx_upload), the refinement, and D2H of the whole refined mesh
    # into pinned host buffers (Engine.download_to -> gdp2d_ctx_download_to).
    # The pinned pools are filled / allocated once, outside the timed region.
    from paper_2007_00324_b200 import PinnedPool
    e2e_steps = a.e2e_steps or a.steps
    e2e_eng = Engine(device)
    pins = []
    for mm in meshes:
        pin_in = PinnedPool(mm.n_vertices, mm.n_triangles, mm.n_subsegments)
        pin_out = PinnedPool(3 * mm.n_vertices, 3 * mm.n_triangles, 3 * mm.n_subsegments)
        pins.append((pin_in.load(mm), pin_in, pin_out))
    for m_in, _, pin_out in pins:        # warm the e2e context (growth, caches)
        e2e_eng.upload(m_in)
        e2e_eng.refine(q)
        e2e_eng.download_to(pin_out)
    e2e_s = []
    e2e_st = 0
    h2d = sum(mesh_bytes(mm) for mm in meshes)
    d2h = 0
    dist.barrier()
    for _ in range(e2e_steps):
        d2h = 0
        t_step = 0.0
        for m_in, _, pin_out in pins:
            t = time.perf_counter()
            e2e_eng.upload(m_in)                  # H2D
            r = e2e_eng.refine(q)
            out = e2e_eng.download_to(pin_out)    # D2H
            t_step += time.perf_counter() - t
            e2e_st += r.steiner_points
            d2h += mesh_bytes(out)
        e2e_s.append(t_step)
    e2e_total = dist.max(sum(e2e_s))
    e2e_value = dist.sum(e2e_st) / e2e_total
    e2e_eng.close()
    del pins

    # ---- e2e through the drop-in C++ shim (reference AoS Mesh, pageable) ----
    dropin = None
    if a.dropin_steps > 0:
        host.time_dropin(meshes[0], cfg["theta"], 1, device)          # warm the cached context
        ds, dst, parts = host.time_dropin(meshes[0], cfg["theta"], a.dropin_steps, device,
                                          parts=True)
        dropin = {"value": dst * a.dropin_steps / ds, "unit": UNIT,
                  "wall_s_per_step": ds / a.dropin_steps, "steps": a.dropin_steps,
                  "path": "gdp2d::refine(cdtref::Mesh&, q, EngineConfig{}) from "
                          "include/gdp2d_cdtref.hpp: the Mesh's element vectors (pageable) to "
                          "gdp2d_refine_aos as they are -- H2D, records converted on the "
                          "device, loop, D2H back into the vectors",
                  "h2d_bytes_per_step": mesh_bytes(meshes[0]), "steiner": dst,
                  "breakdown_s_per_step": parts}

    # ---- the other insertion policies on the same PSLG (reported, not the metric) ----
    modes = None
    if rank == 0 and a.config != 5:
        from paper_2007_00324_b200 import EngineConfig
        gold_m = golden_record(a.config)
        modes = {}
        for name, mode in (("precedence", 2), ("isolated", 0)):
            e = engines[0]
            best = None
            for _ in range(3):
                e.reset()
                r = e.refine(q, EngineConfig(insert_mode=mode))
                best = r if best is None or r.device_seconds < best.device_seconds else best
            modes[name] = {"device_ms": best.device_seconds * 1e3,
                           "steiner_points": best.steiner_points, "batches": len(best.batches),
                           "bad_triangles": best.bad_triangles}
            if gold_m:
                modes[name]["steiner_ratio"] = best.steiner_points / gold_m["steiner_points"]
        modes["note"] = ("gdp2d_params.insert_mode, best of 3 on the bench PSLG; the metric "
                         "uses the default ROLLBACK (the reference's Flip-Flop semantics)")
        engines[0].reset()
        engines[0].refine(q)   # leave the default mode's mesh for the validators

    # ---- roofline: the dominant engine kernel (largest share of the step) ----
    peak, peak_kind = load_peaks()
    kernels = {
        "k_collect_flags": ("Line-3 collect (incremental flags + compaction + candidate scatter)",
                            sum(r.scan_seconds for r in reps), sum(r.scan_bytes for r in reps),
                            sum(r.scan_launches for r in reps)),
        "k_batch_split": ("Lines 5-8a: plan + splits + Lawson flips (persistent)",
                          sum(r.split_seconds for r in reps), sum(r.split_bytes for r in reps),
                          sum(r.split_launches for r in reps)),
        "k_batch_rollback": ("Line 8b: redundancy detection + rollback + Lawson (persistent)",
                             sum(r.rollback_seconds for r in reps),
                             sum(r.rollback_bytes for r in reps),
                             sum(r.rollback_launches for r in reps)),
    }
    traffic_db = {}
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic_db = json.loads(tp.read_text()).get(f"config{a.config}", {})
    per_kernel = {}
    for name, (what, ks, kb, kn) in kernels.items():
        ach = (kb / ks / 1e9) if ks > 0 else None
        per_kernel[name] = {"what": what, "achieved": ach, "frac": (ach / peak) if ach else None,
                            "bytes_per_launch": kb / kn if kn else None,
                            "ms_per_launch": ks / kn * 1e3 if kn else None,
                            "share_of_step": ks / dev_s if dev_s else None,
                            "traffic": traffic_db.get(name)}
    dom = max(per_kernel, key=lambda k: per_kernel[k]["share_of_step"] or 0.0)
    refine_gbs = last.algorithmic_bytes() / last.device_seconds / 1e9
    # device validators on the last timed output (outside the timed region):
    # structure, local CDT, quality, conformity and the min-angle histogram
    validation = engines[-1].validate(q)

    parity = None
    gold = golden_record(a.config) if rank == 0 and a.config != 5 else None
    if gold:
        parity = {
            "reference": "tests/golden/refine_cfg.json (oracle/_ref cdtref::refine, sequential)",
            "same_pslg": gold["pslg_sha"] == sha,
            "reference_steiner": gold["steiner_points"],
            "steiner_ratio": last.steiner_points / gold["steiner_points"],
            "reference_batches": gold["batches"],
            "hist_bin_deg": gold["hist_bin_deg"],
            "min_angle_hist_tv": hist_tv(validation["min_angle_hist"], gold["min_angle_hist"]),
            "mean_min_angle_deg": validation["mean_min_angle_deg"],
            "reference_mean_min_angle_deg": gold["mean_min_angle_deg"],
            "reference_wall_s_in_container": gold["wall_seconds"],
        }
    hist_full = validation.pop("min_angle_hist")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": dev_s_max / a.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, world, sha, seeds[0]),
        "refine_wall_s": dev_s_max / a.steps,
        "steiner_points": last.steiner_points,
        "batches": len(last.batches),
        "quality": {"bad_triangles": last.bad_triangles, "min_angle_deg": last.min_angle_deg},
        "validation": validation,
        "min_angle_hist": {"bin_deg": 0.5, "counts": hist_full},
        "parity": parity,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "wall_s_per_step": e2e_total / e2e_steps,
                "path": "C ABI: gdp2d_ctx_upload (pinned) + gdp2d_ctx_refine + "
                        "gdp2d_ctx_download_to (pinned)"},
        "e2e_dropin": dropin,
        "insert_modes": modes,
        "roofline": {"kernel": dom, "bound": "hbm", "achieved": per_kernel[dom]["achieved"],
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": per_kernel[dom]["frac"], "traffic": per_kernel[dom]["traffic"],
                     "bytes_per_launch": per_kernel[dom]["bytes_per_launch"],
                     "share_of_step": per_kernel[dom]["share_of_step"],
                     "bytes_formula": "DESIGN.md section 3 / include/gdp2d.h gdp2d_report"},
        "roofline_kernels": per_kernel,
        "roofline_refine": {"bytes_alg": last.algorithmic_bytes(), "achieved": refine_gbs,
                            "frac": refine_gbs / peak, "unit": "GB/s",
                            "formula": "SURVEY 8(d) bytes_alg / device refine time"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "host_timed_s": host_s,
        "setup_s": setup_s,
    }

    if rank == 0 and LINE1:
        line["line1_cdt"] = line1_device(device)

    # ---- CPU baseline (rank 0, N = 1 only): the identical PSLG ----
    if world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(cfg, a.config, meshes[0], sha)
    line["native_so_loaded"] = loaded_repo_libs()
    if rank == 0:
        print(json.dumps(line), flush=True)
    for e in engines:
        e.close()
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
