"""Small end-to-end run of every kernel family for compute-sanitizer (tests/test_gpu_sanitizer.py):
integrate (per frame, batched, host frames, colour, projective, trigger), finalize, incremental ESDF,
queries + gradients, surface sampling, pack, the gathered-submap set, import."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_21149_b200 import EsdfSet, Submap  # noqa: E402

dev = torch.device("cuda", 0)
cfg = synth.make_config("tiny", frames=[0, 1, 2, 3])
g = dict(cfg["grid"], max_blocks=2048, esdf_max_distance=0.5)
data = torch.stack([cfg["frames"][k]["data"] for k in range(4)]).to(dev).contiguous()
poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in range(4)])
a = Submap(g, cfg["submaps"][0]["T_world_submap"], 0)
a.integrate(data[0], poses[0], cfg["sensor"])
a.update_esdf()
a.integrate_batch(data[1:3].contiguous(), poses[1:3], cfg["sensor"])
a.integrate_batch_host(data[3:].cpu().contiguous(), poses[3:], cfg["sensor"])
a.update_esdf()
a.finalize_esdf()
pts = (torch.rand((4096, 3), device=dev) * torch.tensor([4.0, 2.0, 1.0], device=dev)).contiguous()
a.query(pts)
a.query_gradient(pts)
a.sample_surface(torch.randint(-2 ** 31, 2 ** 31 - 1, (1024,), device=dev, dtype=torch.int32))
b = Submap(g, cfg["submaps"][0]["T_world_submap"], 0)
b.integrate_until(data, poses, cfg["sensor"], 40)
b.finalize_esdf()
p = Submap(g, cfg["submaps"][0]["T_world_submap"], 0)
p.integrate_projective(data, poses, cfg["sensor"])
gc = dict(g, color=1)
c = Submap(gc, cfg["submaps"][0]["T_world_submap"], 0)
rgb = torch.randint(0, 255, (4, data[0].numel(), 3), device=dev, dtype=torch.uint8)
c.integrate_color(data, rgb, poses, cfg["sensor"])
c.export_color()
pa, pb = a.pack(), b.pack()
buf = torch.cat([pa, torch.zeros((-pa.numel()) % 16, dtype=torch.uint8, device=dev), pb]).contiguous()
es = EsdfSet(buf, [0, pa.numel() + (-pa.numel()) % 16])
es.query(torch.randint(0, 2, (4096,), device=dev, dtype=torch.int32), pts, gradient=True)
bx, D, W, E = a.export()
imp = Submap(g)
imp.import_tsdf(bx, D, W)
imp.finalize_esdf()
torch.cuda.synchronize()
print("sanitize run ok")
