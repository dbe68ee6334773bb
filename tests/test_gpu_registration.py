"""Registration look-ups: ESDF value + gradient queries and
weight-proportional surface sampling, GPU (C-ABI) vs the oracle on the same exported state."""
import numpy as np
import pytest
import torch

import synth
from helpers import gpu_build, gpu_export_sorted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    cfg = synth.make_config("tiny")
    T = synth.pose(synth.rot_zyx(0.3, 0.05, 0.0), [0.5, 0.25, -0.1])
    sm, _ = gpu_build(cfg, list(range(10)), T_ws=T)
    return cfg, sm, gpu_export_sorted(sm)


def test_gradient_parity(built, orc):
    cfg, sm, (b, D, W, E) = built
    s = cfg["grid"]["voxel_size"]
    lo, hi = sm.aabb()
    rng = np.random.default_rng(0)
    xs = rng.uniform(lo * 8 * s, (hi + 1) * 8 * s, (20000, 3))
    xw = (xs @ sm.T_ws[:3, :3].T + sm.T_ws[:3, 3]).astype(np.float32)
    d, g, st = sm.query_gradient(torch.from_numpy(xw).cuda())
    d, g, st = d.cpu().numpy(), g.cpu().numpy(), st.cpu().numpy()
    vo, so, go = orc.query(b, E.astype(np.float64), s, sm.T_ws, xw, gradient=True)
    assert np.array_equal(st, so)
    ok = so == 0
    assert ok.sum() > 300
    fin = ok & np.isfinite(go).all(1)
    assert np.allclose(g[fin], go[fin], atol=1e-4, rtol=1e-5)
    assert np.isnan(g[~ok]).all()
    assert np.allclose(d[so != 2], vo[so != 2], atol=1e-4)


def test_surface_sampling_parity(built, orc):
    cfg, sm, (b, D, W, E) = built
    g = cfg["grid"]
    rng = np.random.default_rng(1)
    u = rng.integers(0, 1 << 32, 50000, dtype=np.uint64).astype(np.uint32)
    xyz, w, tot = sm.sample_surface(torch.from_numpy(u.view(np.int32)).cuda())
    xo, wo, to = orc.sample_surface(b, D.astype(np.float64), W.astype(np.float64), g["site_threshold"],
                                    g["voxel_size"], sm.T_ws, u)
    assert tot == to > 0
    assert np.array_equal(xyz.cpu().numpy().view(np.uint32), xo.view(np.uint32))   # identical picks
    assert np.allclose(w.cpu().numpy(), wo)


def test_surface_sampling_parity_lidar(orc):
    """The same on a LiDAR subset (two configs[1] scans): the block grid spans ~1e5 cells, so the cell-weight
    scan runs over many tiles (three-kernel exact integer scan, registration.cu)."""
    cfg = synth.make_config("lidar", frames=[0, 60])
    sm, _ = gpu_build(cfg, [0, 60], finalize=False)
    b, D, W, _ = gpu_export_sorted(sm)
    lo, hi = sm.aabb()
    assert np.prod(np.asarray(hi) - np.asarray(lo) + 1) > 20000
    g = cfg["grid"]
    rng = np.random.default_rng(2)
    u = rng.integers(0, 1 << 32, 20000, dtype=np.uint64).astype(np.uint32)
    xyz, w, tot = sm.sample_surface(torch.from_numpy(u.view(np.int32)).cuda())
    xo, wo, to = orc.sample_surface(b, D.astype(np.float64), W.astype(np.float64), g["site_threshold"],
                                    g["voxel_size"], sm.T_ws, u)
    assert tot == to > 0
    assert np.array_equal(xyz.cpu().numpy().view(np.uint32), xo.view(np.uint32))
    assert np.allclose(w.cpu().numpy(), wo)
