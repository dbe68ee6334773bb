"""Pins of the oracle's TSDF + Color ("TSDF + Color"; R13).

Reading R13: every update whose unclamped sdf lies inside the truncation band (|sdf| < tau) also adds
w and w * (r, g, b) to the voxel; colour = sum(w c) / sum(w).  References: the parallel-ray plane, where
the band is the closed form |c_z - h| < tau and every ray of a voxel column crosses the whole band, so
each band voxel's colour is the plain mean of the colours of the rays in its column (computed here by
column membership, not by the oracle's traversal); constant colour in -> constant colour out; and
colour weight == TSDF weight on band voxels, 0 elsewhere.
"""
import numpy as np
import pytest

import synth

SENSOR = dict(kind=0, min_range=0.0, max_range=1e9)
GRID = dict(voxel_size=0.1, truncation=0.3, weighting=0, weight_range_floor=0.1, carve=1,
            site_threshold=0.1, max_blocks=1 << 12)


def _plane(orc, weighting=0, seed=3, n=400):
    rng = np.random.default_rng(seed)
    h = 0.4375
    s = orc.OracleSubmap(dict(GRID, weighting=weighting))
    cols = {}
    for k in range(n):
        ix, iy = rng.integers(-12, 12, 2)
        # keep each ray well inside its voxel column (no column-boundary ties)
        x, y = (np.array([ix, iy]) + 0.5 + rng.uniform(-0.35, 0.35, 2)) * 0.1
        H = rng.integers(256, 2048) / 512.0
        T = np.eye(4)
        T[:3, 3] = [x, y, h + H]
        c = np.array([k % 251, (7 * k) % 253, (13 * k + 5) % 256], np.uint8)
        s.integrate_color(np.array([[0.0, 0.0, -H]], np.float32), c[None], T, SENSOR)
        cols.setdefault((int(ix), int(iy)), []).append(c.astype(np.float64))
    return s, h, cols


def _table(s):
    b, D, W = s.export()
    rgb, cw = s.export_color()
    out = {}
    for i in range(b.shape[0]):
        for l in range(512):
            if W[i, l] > 0:
                v = (8 * b[i, 0] + l % 8, 8 * b[i, 1] + (l // 8) % 8, 8 * b[i, 2] + l // 64)
                out[v] = (D[i, l], W[i, l], rgb[i, l], cw[i, l])
    return out


def test_parallel_plane_color_closed_form(orc):
    s, h, cols = _plane(orc)
    t = _table(s)
    n_band = 0
    for (vx, vy, vz), (d, w, rgb, cw) in t.items():
        c = (vz + 0.5) * 0.1
        if abs(c - h) < 0.3:                                   # band voxel: every update is a band update
            n_band += 1
            assert cw == w
            ref = np.mean(cols[(vx, vy)], axis=0)              # every ray of the column crosses the band
            assert np.allclose(rgb, ref, atol=1e-9, rtol=0)
        else:
            assert cw == 0 and (rgb == 0).all()
    assert n_band == 6 * len(cols)                             # vz = 1..6 in every observed column


def test_weighted_band_weight_equals_tsdf_weight(orc):
    s, h, _ = _plane(orc, weighting=1, seed=5)
    for (vx, vy, vz), (d, w, rgb, cw) in _table(s).items():
        c = (vz + 0.5) * 0.1
        assert cw == (pytest.approx(w, rel=1e-12) if abs(c - h) < 0.3 else 0.0)


def test_constant_color_and_bounds_on_lidar(orc):
    cfg = synth.make_config("lidar", frames=[0], lidar_cols=256, color=True)
    f = cfg["frames"][0]
    s = orc.OracleSubmap(cfg["grid"], cfg["submaps"][0]["T_world_submap"])
    const = np.tile(np.array([[17, 200, 93]], np.uint8), (f["rgb"].shape[0], 1))
    s.integrate_color(f["data"].numpy(), const, f["T_world_sensor"], cfg["sensor"])
    _, _, W = s.export()
    rgb, cw = s.export_color()
    has = cw > 0
    assert has.sum() > 1000
    assert np.array_equal(rgb[has], np.tile([17.0, 200.0, 93.0], (int(has.sum()), 1)))
    assert (cw <= W).all() and (cw[~has] == 0).all()
    # textured input: every fused colour lies inside the range of the input colours
    s2 = orc.OracleSubmap(cfg["grid"], cfg["submaps"][0]["T_world_submap"])
    rgb_in = f["rgb"].numpy()
    s2.integrate_color(f["data"].numpy(), rgb_in, f["T_world_sensor"], cfg["sensor"])
    rgb2, cw2 = s2.export_color()
    ok = np.isfinite(f["data"].numpy()).all(1)
    lo, hi = rgb_in[ok].min(0), rgb_in[ok].max(0)
    assert (rgb2[cw2 > 0] >= lo - 1e-9).all() and (rgb2[cw2 > 0] <= hi + 1e-9).all()
    assert np.array_equal(cw2, cw)                              # band membership does not depend on colour
