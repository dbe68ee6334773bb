import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch, synth, oracle
from helpers import gpu_export_sorted
from paper_2410_21149_b200 import Submap
cfg = synth.make_config("lidar", frames=[0, 30, 60, 90])
dev = torch.device("cuda", 0)
sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
for chunk in ([0, 30], [60, 90]):
    for k in chunk:
        sm.integrate(cfg["frames"][k]["data"].to(dev), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
    w = sm.update_esdf()
    b, D, W, E = gpu_export_sorted(sm)
    Eo, _ = oracle.esdf(b, D.astype(np.float64), W.astype(np.float64), 0.2, 0.2)
    fin = np.isfinite(Eo); ex = np.abs(E.astype(np.float64)[fin]) - np.abs(Eo[fin])
    print("waves", w, "finite", fin.sum(), "frac>1e-4", (ex > 1e-4).mean(), "q99", np.quantile(ex, 0.99), "q999", np.quantile(ex, 0.999), "max", ex.max(), "mean", ex.mean())
    # fresh submap with all frames so far: incremental in one shot
sm2 = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
for k in [0, 30, 60, 90]:
    sm2.integrate(cfg["frames"][k]["data"].to(dev), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
w = sm2.update_esdf()
b, D, W, E = gpu_export_sorted(sm2)
Eo, _ = oracle.esdf(b, D.astype(np.float64), W.astype(np.float64), 0.2, 0.2)
fin = np.isfinite(Eo); ex = np.abs(E.astype(np.float64)[fin]) - np.abs(Eo[fin])
print("one-shot waves", w, "frac>1e-4", (ex > 1e-4).mean(), "q99", np.quantile(ex, 0.99), "max", ex.max())
