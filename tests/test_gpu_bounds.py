"""The library built with CVX_BOUNDS=1 (device-side index checks on the hot kernels' global writes and
reductions: dense-window and pool accumulator addresses, ray start inside the launch's block box, dense
fold slots, ESDF ring-stack depth / refill ranges / line outputs, pass-x rows and plane slots; a failed
check prints and traps) on a small run of every kernel family (tools/sanitize_tiny.py) and on the bench's
own LiDAR / ESDF-stress shapes (tools/bounds_lidar.py).  compute-sanitizer is closed on some GPU pools
(tests/test_gpu_sanitizer.py skips there); this is the library's own bounds evidence."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bounds_lib():
    from paper_2410_21149_b200 import build
    return build.build_bounds()


@pytest.mark.parametrize("script", ["sanitize_tiny.py", "bounds_lidar.py"])
def test_bounds_checked_build_runs_clean(bounds_lib, script):
    env = dict(os.environ, CVX_LIB_PATH=bounds_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", script)], capture_output=True, text=True,
                       timeout=1200, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "run ok" in out and "bounds check failed" not in out, out[-3000:]
