"""Hash-table stress test (Fig. 7) at CI size: the library's own
`hash_activate` / `hash_find` device functions (microbench/hash_stress.cu) on ~1 M random distinct block
keys at load factors 0.5 and 0.9 — every key gets a distinct slot in [0, n), re-activation and lookup
return the same slot, no capacity / hash-full error."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_hash_stress_ci(tmp_path):
    exe = str(tmp_path / "hash_stress")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", exe,
                           os.path.join(ROOT, "microbench", "hash_stress.cu")])
    out = subprocess.run([exe, "21", "0.5", "20", "0.9"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(rows) == 2
    for r in rows:
        assert r["ok"] and r["errors"] == 0 and r["blocks"] == r["keys"]
    assert rows[0]["mean_probe"] < rows[1]["mean_probe"]     # linear probing: longer chains at higher load
