"""Full-size checks of the projection-mapping integrator on BASELINE.json configs[2]:
the first submap (100 synthetic 640x480 depth frames, 5 cm voxels) in the launch configuration
`bench.py --workload rgbd` times (one integrate_projective call of 100 frames).  Sampled outputs are
checked against the oracle voxel by voxel; the rest by properties that hold at any size.
"""
import numpy as np
import pytest
import torch

import synth
from helpers import TOL_D, TOL_W, gpu_export_sorted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rgbd():
    dev = torch.device("cuda", 0)
    cfg = synth.make_config("rgbd", frames=list(range(100)), device=dev)
    depth = torch.stack([cfg["frames"][k]["data"] for k in range(100)]).contiguous()
    poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in range(100)])
    return cfg, depth, poses


def _proj(cfg, depth, poses, chunk):
    from paper_2410_21149_b200 import Submap
    sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    st = None
    for c in range(0, depth.shape[0], chunk):
        st = sm.integrate_projective(depth[c:c + chunk], poses[c:c + chunk], cfg["sensor"], stats=True)
    return sm, st


def test_fullsize_projective_properties(rgbd):
    cfg, depth, poses = rgbd
    sm, st = _proj(cfg, depth, poses, 100)
    b, D, W, _ = gpu_export_sorted(sm)
    assert st["rays_in"] == 100 * 640 * 480 and b.shape[0] > 500
    assert W.astype(np.float64).sum() == st["voxel_updates"]          # constant weights: one unit per update
    # frame-by-frame calls (birth frames never used) == one call (birth frames) bit for bit
    s1, _ = _proj(cfg, depth, poses, 1)
    b1, D1, W1, _ = gpu_export_sorted(s1)
    assert np.array_equal(b1, b)
    assert np.array_equal(D1.view(np.uint32), D.view(np.uint32)) and np.array_equal(W1.view(np.uint32), W.view(np.uint32))
    # ALLOCATE is the raycaster's
    from paper_2410_21149_b200 import Submap
    r = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    r.integrate_batch(depth, poses, cfg["sensor"])
    assert np.array_equal(gpu_export_sorted(r)[0], b)


def test_fullsize_projective_sampled_vs_oracle(rgbd, orc):
    cfg, depth, poses = rgbd
    sm, _ = _proj(cfg, depth, poses, 100)
    b, D, W, _ = gpu_export_sorted(sm)
    s0, _ = _proj(cfg, depth[:1], poses[:1], 1)              # blocks existing from frame 0 on
    b0 = gpu_export_sorted(s0)[0]
    rows = {tuple(x) for x in b0.tolist()}
    idx = np.array([i for i, x in enumerate(b.tolist()) if tuple(x) in rows])
    rng = np.random.default_rng(7)
    pick_b = rng.choice(idx, 4096)
    pick_l = rng.integers(0, 512, 4096)
    bb = b[pick_b]
    vox = np.stack([8 * bb[:, 0] + pick_l % 8, 8 * bb[:, 1] + (pick_l // 8) % 8, 8 * bb[:, 2] + pick_l // 64], 1)
    swd, sw = orc.project_voxels(cfg["grid"], cfg["submaps"][0]["T_world_submap"], depth.cpu().numpy(), poses,
                                 cfg["sensor"], vox)
    Wg, Dg = W[pick_b, pick_l].astype(np.float64), D[pick_b, pick_l].astype(np.float64)
    assert np.array_equal(Wg > 0, sw > 0)
    obs = sw > 0
    assert obs.sum() > 500
    assert np.abs(Wg[obs] - sw[obs]).max() <= TOL_W * max(1.0, sw.max())
    assert np.abs(Dg[obs] - swd[obs] / sw[obs]).max() <= TOL_D
