"""Bounds-checked run on the bench's own workloads (tests/test_gpu_bounds.py): 20 configs[1] scans through
the dense-window path and through its device-side fallback, the exact ESDF of both, 1 M queries, and a
small configs[4]-style import + ESDF (ring line kernels at 2 cm)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21149_b200 import Submap  # noqa: E402

dev = torch.device("cuda", 0)
cfg = synth.make_config("lidar", frames=list(range(20)), device=dev)
data = torch.stack([cfg["frames"][k]["data"] for k in range(20)]).contiguous()
poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in range(20)])
for blocks in (None, "1000"):
    if blocks:
        os.environ["CVX_DENSE_BLOCKS"] = blocks      # forces the device-side fallback (box > buffer)
    sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    sm.integrate_batch(data, poses, cfg["sensor"])
    sm.finalize_esdf()
    q = (torch.rand((1 << 20, 3), device=dev) * 60 - 30).contiguous()
    sm.query(q)
    torch.cuda.synchronize()
os.environ.pop("CVX_DENSE_BLOCKS", None)
g = dict(voxel_size=0.02, truncation=0.06, site_threshold=0.02, max_blocks=40000)
im = Submap(g, np.eye(4), 0)
for b, D, W in synth.scenes.esdf_stress_blocks(extent=(4.0, 4.0, 1.0), device=dev):
    im.import_tsdf(b, D, W)
im.finalize_esdf()
torch.cuda.synchronize()
print("bounds run ok")
