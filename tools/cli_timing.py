"""Wall time of gdp2d_cli on a BASELINE config-2 PSLG written as .poly, per
I/O mode (host path vs --device-cdt / --device-io).  GPU box only."""
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from paper_2007_00324_b200 import host  # noqa: E402
from test_dropin_cli import CLI, write_poly  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    out = Path("gpurun_out") if Path("gpurun_out").exists() else Path("/tmp")
    poly = out / "cli_in.poly"
    pts, segs = host.generate_pslg(n, n // 10, "uniform", 20261017)
    write_poly(poly, pts, segs)
    for flags in ([], ["--device-cdt"], ["--device-io"], ["--device-cdt", "--device-io"]):
        t0 = time.perf_counter()
        r = subprocess.run([str(CLI), str(poly), "--out", str(out / "cli_out")] + flags,
                           capture_output=True, text=True)
        dt = time.perf_counter() - t0
        print(f"{' '.join(flags) or '(host path)':28s} rc={r.returncode} wall {dt:.2f} s  "
              f"{r.stdout.strip()}", flush=True)
    for p in out.glob("cli_*"):
        p.unlink()


if __name__ == "__main__":
    main()
