"""Serial per-kernel breakdown of the MAV workload (configs[3]): every submap built one after another on one
builder with serialised profiling (solo kernel times), summed over the 40 submaps; plus the dense AABB
sizes of the submaps.  usage: python tools/diag_mav.py [n_submaps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2410_21149_b200 as cvx  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = synth.make_config("mav", frames=[], device=dev)
subs = cfg["submaps"][:n]
frames = sorted(k for s in subs for k in s["frames"])
cf = synth.make_config("mav", frames=frames, device=dev)
b = cvx.Submap(cfg["grid"], subs[0]["T_world_submap"], 0)
tot = {}
vox = []
for rep in range(2):
    for s in subs:
        d = torch.stack([cf["frames"][k]["data"] for k in s["frames"]]).contiguous()
        p = np.stack([cf["frames"][k]["T_world_sensor"] for k in s["frames"]])
        b.reset(s["T_world_submap"])
        b.profile(rep == 1, serialize=True)
        b.integrate_batch(d, p, cfg["sensor"])
        b.finalize_esdf()
        b.pack()
        torch.cuda.synchronize()
        if rep == 1:
            for k, v in b.profile_report().items():
                tot[k] = tot.get(k, 0.0) + v["ms"]
            lo, hi = b.aabb()
            vox.append(int(np.prod((np.asarray(hi) - np.asarray(lo) + 1) * 8)))
        b.profile(False)
print({k: round(v, 2) for k, v in sorted(tot.items(), key=lambda x: -x[1])})
print("sum", round(sum(tot.values()), 2), "ms; dense AABB voxels per submap: mean %.3g max %.3g" % (np.mean(vox), np.max(vox)))
