"""Calibrate the timed reference arm (the numpy port oracle/cpu_baseline.py,
which is what bench.py --impl reference runs on the GPU box, where
/root/reference does not exist) against the REAL reference timed here:
`distfno scale --transport proc` (d/cli.py:158-191, d/bench.py:359-400) with
P worker processes on this container's cores, versus the port with the same
decomposition on the same cores.  Writes profiles/r02_reference_calibration.json.
Runs only where /root/reference exists (this container).
usage: python tools/calibrate_reference_arm.py [grid] [P] [iters]"""
import json
import os
import platform
import re
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import cpu_baseline as CB  # noqa: E402


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main(grid="32,32,32,16", P=8, iters=2):
    g = tuple(int(v) for v in grid.split(","))
    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src", PYTHONDONTWRITEBYTECODE="1",
               OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1")
    out = tempfile.mktemp(suffix=".csv")
    cmd = [sys.executable, "-m", "distfno.cli", "scale", "--workers", str(P), "--mode", "strong", "--grid", grid,
           "--modes", "8,8,8,8", "--channels", "20", "--blocks", "4", "--dtype", "f32", "--activation", "gelu",
           "--iters", str(iters), "--transport", "proc", "--out", out]
    t0 = time.time()
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=tempfile.gettempdir())
    wall = time.time() - t0
    m = re.search(r"forward ([\d.]+) ms, fwd\+bwd ([\d.]+) ms", r.stdout)
    if not m:
        raise SystemExit(r.stdout + r.stderr)
    ref_fwd, ref_fb = float(m.group(1)) / 1e3, float(m.group(2)) / 1e3
    per_step, job = CB.measure(g, 20, (8, 8, 8, 8), 4, P, P, steps=iters)
    port_fb = min(job)
    res = {
        "what": "real reference (distfno scale --transport proc) vs the timed numpy port, same decomposition, same cores",
        "grid": list(g), "channels": 20, "blocks": 4, "modes": [8, 8, 8, 8], "P": P, "cores": os.cpu_count(),
        "cpu_model": cpu_model(),
        "reference_cmd": " ".join(cmd[1:]),
        "reference_fwd_s": ref_fwd, "reference_fwd_bwd_s": ref_fb, "reference_wall_s": round(wall, 1),
        "port_fwd_bwd_s": port_fb,
        "reference_over_port": ref_fb / port_fb,
        "note": "ratio > 1 means the real reference is slower than the port, i.e. the bench's reference arm "
                "(the port) overstates the reference's throughput by this factor",
    }
    print(json.dumps(res, indent=1))
    (ROOT / "profiles").mkdir(exist_ok=True)
    name = f"r02_reference_calibration_{'x'.join(map(str, g))}_P{P}.json"
    (ROOT / "profiles" / name).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "32,32,32,16", int(a[1]) if len(a) > 1 else 8, int(a[2]) if len(a) > 2 else 2)
