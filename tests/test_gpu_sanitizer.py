"""compute-sanitizer on a small run of every kernel family (tools/sanitize_tiny.py): memcheck (out of
bounds / misaligned accesses, including the hash's publish-and-spin protocol and the cp.async slot
prefetch), racecheck (shared-memory hazards: TMA-staged ESDF tiles, pass-x plane staging, the incremental
window), synccheck (barrier / warp-sync misuse).  0 errors required."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_tiny.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT)
    out = r.stdout + r.stderr
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log") if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
              else os.devnull, "w") as f:
        f.write(out)
    if "closed on this pool" in out:   # the GPU pool replaced compute-sanitizer with a refusal stub
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert "sanitize run ok" in out, out[-3000:]
    clean = "ERROR SUMMARY: 0 errors" in out or "SUMMARY: 0 hazards displayed (0 errors" in out
    assert r.returncode == 0 and clean, out[-3000:]
