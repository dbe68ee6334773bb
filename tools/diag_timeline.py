"""Phase timeline of one bench step (configs[1]) with CUDA events on the caller's stream."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_21149_b200 as cvx  # noqa: E402

dev = torch.device("cuda", 0)
cfg, data, poses = bench.make_workload(0, dev)
sm = cvx.Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
q = torch.rand((1 << 20, 3), device=dev) * 50
qo = torch.empty(1 << 20, device=dev)
qs = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
batch = int(os.environ.get("BATCH", "200"))


def step(ev=None):
    def mark():
        if ev is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev.append(e)
    mark()
    sm.reset()
    mark()
    for c in range(0, 200, batch):
        sm.integrate_batch(data[c:c + batch], poses[c:c + batch], cfg["sensor"])
    mark()
    sm.finalize_esdf()
    mark()
    sm.query(q, qo, qs)
    mark()


for _ in range(3):
    step()
torch.cuda.synchronize()
for prof in (False, True):
    sm.profile(prof)
    evs = []
    for _ in range(5):
        ev = []
        step(ev)
        evs.append(ev)
    torch.cuda.synchronize()
    ph = np.array([[a.elapsed_time(b) for a, b in zip(ev[:-1], ev[1:])] for ev in evs])
    tot = np.array([ev[0].elapsed_time(ev[-1]) for ev in evs])
    gaps = [evs[i][-1].elapsed_time(evs[i + 1][0]) for i in range(len(evs) - 1)]
    print(f"profile={prof}: reset {ph[:,0].mean():.3f} integrate {ph[:,1].mean():.3f} finalize {ph[:,2].mean():.3f} "
          f"query {ph[:,3].mean():.3f} total {tot.mean():.3f} inter-step gap {np.mean(gaps):.3f} ms")
    if prof:
        print({k: round(v, 3) for k, v in sm.profile_report().items()})
    sm.profile(False)
