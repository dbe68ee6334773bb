"""GPU parity of the projection-mapping integrator (R14).

libcvx `cvx_integrate_projective` (through the C-ABI) vs the oracle's `orc_integrate_projective` on the
same seeded depth frames.  Bar: block sets and observed sets bit-exact (every decision — z > 0, nearest
pixel, range, occlusion — is taken in the same fp64/fp32 operation order on both sides), projective
update counts exact, |dD| <= 1e-4 m, |dW| <= 1e-3 max(1, W); batches equal frame-by-frame calls bit for
bit; the block set equals the raycast integrator's (shared ALLOCATE).
"""
import numpy as np
import pytest
import torch

import synth
from helpers import assert_tsdf_parity, gpu_export_sorted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    return synth.make_config("tiny")


def _gpu(cfg, frames, grid=None, T_ws=None, batch=True):
    from paper_2410_21149_b200 import Submap
    g = dict(cfg["grid"] if grid is None else grid)
    T = cfg["submaps"][0]["T_world_submap"] if T_ws is None else T_ws
    sm = Submap(g, T, 0)
    dev = torch.device("cuda", 0)
    if batch:
        depth = torch.stack([cfg["frames"][k]["data"] for k in frames]).to(dev)
        poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in frames])
        st = sm.integrate_projective(depth, poses, cfg["sensor"], stats=True)
    else:
        for k in frames:
            st = sm.integrate_projective(cfg["frames"][k]["data"].to(dev).contiguous(),
                                         cfg["frames"][k]["T_world_sensor"][None], cfg["sensor"], stats=True)
    return sm, st


def _orc(orc, cfg, frames, grid=None, T_ws=None):
    g = dict(cfg["grid"] if grid is None else grid)
    T = cfg["submaps"][0]["T_world_submap"] if T_ws is None else T_ws
    o = orc.OracleSubmap(g, T)
    sts = [o.integrate_projective(cfg["frames"][k]["data"].numpy(), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
           for k in frames]
    return o, sts


def test_tiny_projective_parity_and_counts(tiny, orc):
    frames = list(range(10))
    sm, st = _gpu(tiny, frames)
    o, sts = _orc(orc, tiny, frames)
    rep = assert_tsdf_parity(gpu_export_sorted(sm), o.export())
    assert rep["observed"] > 5000
    for key in ("rays_in", "rays_used", "skipped_invalid", "skipped_range", "voxel_updates"):
        assert st[key] == sum(s[key] for s in sts), key
    _, _, W, _ = gpu_export_sorted(sm)
    assert W.astype(np.float64).sum() == st["voxel_updates"]     # constant weights: one unit per update


@pytest.mark.parametrize("weighting,carve", [(1, 1), (0, 0), (1, 0)])
def test_tiny_projective_modes(tiny, orc, weighting, carve):
    g = dict(tiny["grid"], weighting=weighting, carve=carve)
    frames = [0, 4, 9]
    T_ws = synth.scenes.pose(synth.scenes.rot_zyx(0.3, 0.1, -0.05), [0.7, -0.4, 0.2])   # non-trivial submap pose
    sm, _ = _gpu(tiny, frames, grid=g, T_ws=T_ws)
    o, _ = _orc(orc, tiny, frames, grid=g, T_ws=T_ws)
    assert_tsdf_parity(gpu_export_sorted(sm), o.export())


def test_batch_equals_per_frame_bitexact(tiny):
    frames = list(range(10))
    a, _ = _gpu(tiny, frames, batch=True)
    b, _ = _gpu(tiny, frames, batch=False)
    ea, eb = gpu_export_sorted(a), gpu_export_sorted(b)
    assert np.array_equal(ea[0], eb[0])
    assert np.array_equal(ea[1].view(np.uint32), eb[1].view(np.uint32))
    assert np.array_equal(ea[2].view(np.uint32), eb[2].view(np.uint32))


def test_block_set_equals_raycast(tiny):
    from helpers import gpu_build
    frames = list(range(10))
    a, _ = _gpu(tiny, frames)
    r, _ = gpu_build(tiny, frames, batch=True, finalize=False)
    assert np.array_equal(gpu_export_sorted(a)[0], gpu_export_sorted(r)[0])


def test_rgbd_subset_projective_parity(orc):
    cfg = synth.make_config("rgbd", frames=[0, 23, 61])
    sm, st = _gpu(cfg, [0, 23, 61])
    o, sts = _orc(orc, cfg, [0, 23, 61])
    rep = assert_tsdf_parity(gpu_export_sorted(sm), o.export())
    assert rep["blocks"] > 500
    assert st["voxel_updates"] == sum(s["voxel_updates"] for s in sts)


def test_more_frames_than_one_launch(tiny, orc):
    # 130 frames > kMaxBatch (128): two launches, birth counts per launch
    frames = [k % 10 for k in range(130)]
    sm, st = _gpu(tiny, frames)
    o, sts = _orc(orc, tiny, frames)
    assert_tsdf_parity(gpu_export_sorted(sm), o.export())
    assert st["voxel_updates"] == sum(s["voxel_updates"] for s in sts)


def test_projective_then_esdf_and_errors(tiny):
    from paper_2410_21149_b200 import Submap, CvxError
    sm, _ = _gpu(tiny, [0, 1, 2])
    sm.finalize_esdf()
    _, _, _, E = gpu_export_sorted(sm)
    assert np.isfinite(E).sum() > 1000
    lidar = dict(kind=2, width=8, height=4, min_range=0.1, max_range=10.0)
    s2 = Submap(tiny["grid"], np.eye(4), 0)
    with pytest.raises(CvxError):
        s2.integrate_projective(torch.zeros((1, 4, 8), device="cuda"), np.eye(4)[None], lidar)
