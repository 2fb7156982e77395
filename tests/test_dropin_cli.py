"""The drop-in C++ path: the reference CLI's run_one with cdtref::refine
swapped for gdp2d::refine (include/gdp2d_cdtref.hpp, lib/gdp2d_cli).  CPU
tests check it links against libgdp2d.so and keeps cdtref.cpp's exit codes;
the GPU test refines a .poly end to end and reads the .node/.ele back."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2007_00324_b200" / "lib" / "gdp2d_cli"


def write_poly(path: Path, pts: np.ndarray, segs: np.ndarray) -> None:
    lines = [f"{len(pts)} 2 0 0"]
    lines += [f"{i} {x!r} {y!r}" for i, (x, y) in enumerate(pts.tolist())]
    lines.append(f"{len(segs)} 0")
    lines += [f"{i} {a} {b}" for i, (a, b) in enumerate(segs.tolist())]
    lines.append("0")
    path.write_text("\n".join(lines) + "\n")


def test_cli_usage_and_input_errors(built, tmp_path):
    assert CLI.exists()
    assert subprocess.run([str(CLI)], capture_output=True).returncode == 2
    assert subprocess.run([str(CLI), str(tmp_path / "missing.poly")],
                          capture_output=True).returncode == 2
    bad = tmp_path / "bad.poly"
    bad.write_text("3 2 0 0\n0 0 0\n1 1 0\n")          # truncated vertex list
    assert subprocess.run([str(CLI), str(bad)], capture_output=True).returncode == 2


def test_cli_without_gpu_fails_loudly(built, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from gdp2d_testlib import unit_square
    pts, segs = unit_square()
    poly = tmp_path / "sq.poly"
    write_poly(poly, pts, segs)
    r = subprocess.run([str(CLI), str(poly)], capture_output=True, text=True)
    assert r.returncode == 4, r.stderr           # engine error, never a CPU fallback
    assert "engine error" in r.stderr


@pytest.mark.gpu
def test_cli_refines_poly(built, tmp_path):
    from paper_2007_00324_b200 import host
    pts, segs = host.generate_pslg(20_000, 2_000, "uniform", 4)
    poly = tmp_path / "in.poly"
    write_poly(poly, pts, segs)
    r = subprocess.run([str(CLI), str(poly), "--theta", "20.704811054635428", "--out",
                        str(tmp_path / "out")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    kv = dict(t.split("=") for t in r.stdout.split())
    assert int(kv["bad_triangles"]) == 0
    assert float(kv["min_angle_deg"]) >= 20.704811054635428 - 1e-9
    node = (tmp_path / "out.node").read_text().splitlines()
    ele = (tmp_path / "out.ele").read_text().splitlines()
    nv = int(node[0].split()[0])
    nt = int(ele[0].split()[0])
    assert nv == int(kv["output_points"]) == len(node) - 1
    assert nv - 20_000 == int(kv["steiner_points"])
    tri = np.array([list(map(int, l.split()[1:])) for l in ele[1:]])
    assert tri.shape == (nt, 3) and tri.max() < nv


@pytest.mark.gpu
def test_cli_device_cdt(built, tmp_path):
    """--device-cdt: Line 1 on the GPU too (gdp2d::build_cdt); same quality bar,
    and a PSLG the reference rejects (duplicate point) still exits 2."""
    from paper_2007_00324_b200 import host
    pts, segs = host.generate_pslg(20_000, 2_000, "gaussian", 6)
    poly = tmp_path / "in.poly"
    write_poly(poly, pts, segs)
    r = subprocess.run([str(CLI), str(poly), "--device-cdt", "--out", str(tmp_path / "out")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    kv = dict(t.split("=") for t in r.stdout.split())
    assert int(kv["bad_triangles"]) == 0 and int(kv["steiner_points"]) > 0
    assert (tmp_path / "out.ele").exists()


@pytest.mark.gpu
def test_cli_device_io_same_bytes(built, tmp_path):
    """--device-io (device validators, device compaction, parallel text) writes
    the same .node/.ele bytes as the host path (write_node_ele) for the same
    refinement, with and without the device CDT."""
    from paper_2007_00324_b200 import host
    pts, segs = host.generate_pslg(30_000, 3_000, "uniform", 8)
    poly = tmp_path / "in.poly"
    write_poly(poly, pts, segs)
    outs = {}
    for tag, flags in {"host": [], "dio": ["--device-io"], "dcdt": ["--device-cdt"],
                       "dcdt_dio": ["--device-cdt", "--device-io"]}.items():
        r = subprocess.run([str(CLI), str(poly), "--out", str(tmp_path / tag)] + flags,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, (tag, r.stdout + r.stderr)
        outs[tag] = ((tmp_path / f"{tag}.node").read_bytes(), (tmp_path / f"{tag}.ele").read_bytes(),
                     r.stdout.split("wall_seconds")[0])
    assert outs["host"][:2] == outs["dio"][:2] and outs["host"][2] == outs["dio"][2]
    assert outs["dcdt"][:2] == outs["dcdt_dio"][:2]
