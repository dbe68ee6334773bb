"""Pins of the oracle's projection-mapping integrator (R14).

P:L104: "projects voxels in the visual field of view into the depth image and computes their distance
from the difference between the voxel centre and the depth value in the image"; "associating
it with the nearest pixel".  References used (none of them re-runs the oracle's own formula):
  * a fronto-parallel wall seen by a camera with an exactly representable 90-degree yaw: closed form
    D = min(h - z_v, tau) with z_v the voxel centre's depth along the WORLD optical axis, occluded
    voxels (h - z_v < -tau) unobserved, W = frames;
  * the nearest-pixel association checked in exact rational arithmetic (fractions) against a depth
    image whose value encodes (px, py) differently per axis (catches u/v transposition, floor vs round,
    half-pixel offsets);
  * the inverse-square weight from the PIXEL's ray length, closed form on the wall;
  * the block set equals the raycast integrator's (ALLOCATE is shared);
  * same frame twice (weights double), frame-order invariance, band mode, range filter.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import synth

S = 0.125          # dyadic voxel size: voxel centres exact
TAU = 0.375
CAM = dict(kind=1, width=64, height=48, fx=32.0, fy=32.0, cx=31.5, cy=23.5, min_range=0.05, max_range=20.0)


def _grid(**kw):
    g = dict(voxel_size=S, truncation=TAU, weighting=0, weight_range_floor=0.1, carve=1, site_threshold=S,
             max_blocks=1 << 14)
    g.update(kw)
    return g


def _pose_yaw90(o):
    """Camera looking along world +y (exact 90-degree yaw of the +x-looking camera; entries 0 / +-1)."""
    return synth.scenes.camera_pose(o, np.pi / 2, 0.0).round(15)


def _table(sm):
    b, D, W = sm.export()
    vox = []
    for i in range(b.shape[0]):
        l = np.arange(512)
        v = np.stack([8 * b[i, 0] + l % 8, 8 * b[i, 1] + (l // 8) % 8, 8 * b[i, 2] + l // 64], 1)
        vox.append(v)
    V = np.concatenate(vox) if vox else np.zeros((0, 3), np.int64)
    return b, V, D.reshape(-1), W.reshape(-1)


def _cam_coords(V, T_wc):
    """Exact camera-frame coordinates of the voxel centres (world = submap frame, rational arithmetic)."""
    R = [[Fr(float(T_wc[i, j])) for j in range(3)] for i in range(3)]
    o = [Fr(float(T_wc[i, 3])) for i in range(3)]
    out = []
    for v in V:
        c = [(Fr(int(v[k])) + Fr(1, 2)) * Fr(S) - o[k] for k in range(3)]
        out.append([R[0][i] * c[0] + R[1][i] * c[1] + R[2][i] * c[2] for i in range(3)])
    return out


def _pixel(x):
    """Nearest pixel (pixel centres at integers, Q24) in exact arithmetic; None outside the image or
    within 1e-9 of a pixel boundary (where fp64 rounding may decide either way)."""
    if x[2] <= 0:
        return None
    uh = Fr(CAM["fx"]) * x[0] / x[2] + Fr(CAM["cx"]) + Fr(1, 2)
    wh = Fr(CAM["fy"]) * x[1] / x[2] + Fr(CAM["cy"]) + Fr(1, 2)
    for a, n in ((uh, CAM["width"]), (wh, CAM["height"])):
        f = a - (a.numerator // a.denominator)
        if f < Fr(1, 10**9) or f > 1 - Fr(1, 10**9):
            return "edge"
        if a < 0 or a >= n:
            return None
    return int(uh), int(wh)


def test_wall_closed_form_rotated_camera(orc):
    h = 2.0
    T = _pose_yaw90([0.3125, -0.0625, 1.0625])
    depth = np.full((48, 64), h, np.float32)
    sm = orc.OracleSubmap(_grid())
    st = sm.integrate_projective(depth, T, CAM)
    sm.integrate_projective(depth, T, CAM)
    _, V, D, W = _table(sm)
    axis = T[:3, 2]                              # world optical axis (camera z)
    assert np.array_equal(np.abs(axis), [0, 1, 0])
    X = _cam_coords(V, T)
    n_obs = n_occ = 0
    for i, x in enumerate(X):
        px = _pixel(x)
        if px == "edge":
            continue
        zw = ((V[i] + 0.5) * S - T[:3, 3]) @ axis   # depth along the world optical axis
        assert float(x[2]) == zw
        if px is None or h - zw < -TAU:
            assert W[i] == 0.0, (V[i], px, zw)
            n_occ += px is not None
        else:
            assert W[i] == 2.0
            assert D[i] == min(h - zw, TAU)        # projective (along-axis) distance, clamped at +tau
            n_obs += 1
    assert n_obs > 1000 and n_occ > 100
    assert st["voxel_updates"] * 2 == int(W.sum())


def test_nearest_pixel_association_exact(orc):
    # depth encodes the pixel: m = 1.5 + 0.01 px + 0.003 py (x and y steps differ)
    py, px = np.mgrid[0:48, 0:64]
    depth = (1.5 + 0.01 * px + 0.003 * py).astype(np.float32)
    T = _pose_yaw90([0.0625, 0.0, 1.0])
    sm = orc.OracleSubmap(_grid())
    sm.integrate_projective(depth, T, CAM)
    _, V, D, W = _table(sm)
    X = _cam_coords(V, T)
    checked = 0
    for i, x in enumerate(X):
        p = _pixel(x)
        if p is None or p == "edge":
            continue
        sdf = float(depth[p[1], p[0]]) - float(x[2])
        if sdf < -TAU:
            assert W[i] == 0.0
            continue
        assert W[i] == 1.0
        assert D[i] == pytest.approx(min(sdf, TAU), abs=1e-12)
        checked += 1
    assert checked > 1000


def test_inverse_square_weight_uses_pixel_ray_length(orc):
    h = 2.5
    T = _pose_yaw90([0.0, 0.0, 1.0])
    depth = np.full((48, 64), h, np.float32)
    sm = orc.OracleSubmap(_grid(weighting=1))
    sm.integrate_projective(depth, T, CAM)
    _, V, D, W = _table(sm)
    X = _cam_coords(V, T)
    checked = 0
    for i, x in enumerate(X):
        p = _pixel(x)
        if p is None or p == "edge" or h - float(x[2]) < -TAU:
            continue
        L = h * np.sqrt(1 + ((p[0] - 31.5) / 32.0) ** 2 + ((p[1] - 23.5) / 32.0) ** 2)
        assert W[i] == pytest.approx(1.0 / L**2, rel=1e-6)   # fp32 pixel point (O2)
        checked += 1
    assert checked > 1000


def test_block_set_equals_raycast_allocation(orc):
    cfg = synth.make_config("tiny", frames=[0, 5])
    a = orc.OracleSubmap(cfg["grid"])
    b = orc.OracleSubmap(cfg["grid"])
    for k in (0, 5):
        fr = cfg["frames"][k]
        sa = a.integrate(fr["data"].numpy(), fr["T_world_sensor"], cfg["sensor"])
        sb = b.integrate_projective(fr["data"].numpy(), fr["T_world_sensor"], cfg["sensor"])
        for key in ("rays_in", "rays_used", "skipped_invalid", "skipped_range", "new_blocks", "total_blocks"):
            assert sa[key] == sb[key], key
    ba, _, Wa = a.export()
    bb, _, Wb = b.export()
    assert np.array_equal(ba, bb)
    assert (Wb > 0).sum() > 0


def test_same_frame_twice_and_order_invariance(orc):
    cfg = synth.make_config("tiny", frames=[1, 7])
    f1, f7 = cfg["frames"][1], cfg["frames"][7]
    a = orc.OracleSubmap(cfg["grid"])
    a.integrate_projective(f1["data"].numpy(), f1["T_world_sensor"], cfg["sensor"])
    _, D1, W1 = a.export()
    a.integrate_projective(f1["data"].numpy(), f1["T_world_sensor"], cfg["sensor"])
    _, D2, W2 = a.export()
    assert np.array_equal(W2, 2 * W1) and np.allclose(D1, D2, atol=1e-12)
    # once the block set is fixed (both submaps first take f1, f7), the sums commute: f1 f7 == f7 f1
    x = orc.OracleSubmap(cfg["grid"])
    y = orc.OracleSubmap(cfg["grid"])
    for sm, order in ((x, (f1, f7, f1, f7)), (y, (f1, f7, f7, f1))):
        for fr in order:
            sm.integrate_projective(fr["data"].numpy(), fr["T_world_sensor"], cfg["sensor"])
    bx, Dx, Wx = x.export()
    by, Dy, Wy = y.export()
    assert np.array_equal(bx, by) and np.array_equal(Wx, Wy)
    assert np.allclose(Dx, Dy, atol=1e-12)


def test_band_mode_and_range_filter(orc):
    h = 2.0
    T = _pose_yaw90([0.0, 0.0, 1.0])
    depth = np.full((48, 64), h, np.float32)
    band = orc.OracleSubmap(_grid(carve=0))
    band.integrate_projective(depth, T, CAM)
    _, V, D, W = _table(band)
    obs = W > 0
    assert obs.sum() > 100 and np.all(np.abs(D[obs]) <= TAU)
    X = _cam_coords(V[obs], T)
    assert all(abs(h - float(x[2])) <= TAU for x in X)
    # every pixel beyond max_range: no allocation, no update
    far = orc.OracleSubmap(_grid())
    st = far.integrate_projective(depth, T, dict(CAM, max_range=1.5))
    assert st["skipped_range"] == 64 * 48 and far.num_blocks() == 0 and st["voxel_updates"] == 0


def test_project_voxels_hook_matches_integration(orc):
    # the sampled-check hook (per-voxel sums over all frames) equals whole-submap integration for voxels
    # whose block exists from the first frame on
    cfg = synth.make_config("tiny", frames=[0, 3, 6])
    fr = [cfg["frames"][k] for k in (0, 3, 6)]
    first = orc.OracleSubmap(cfg["grid"])
    first.integrate_projective(fr[0]["data"].numpy(), fr[0]["T_world_sensor"], cfg["sensor"])
    b0, _, _ = first.export()
    full = orc.OracleSubmap(cfg["grid"])
    for f in fr:
        full.integrate_projective(f["data"].numpy(), f["T_world_sensor"], cfg["sensor"])
    b, D, W = full.export()
    keep = np.array([any((bb == x).all() for x in b0) for bb in b])
    l = np.arange(512)
    vox = np.concatenate([np.stack([8 * bb[0] + l % 8, 8 * bb[1] + (l // 8) % 8, 8 * bb[2] + l // 64], 1) for bb in b[keep]])
    depth = np.stack([f["data"].numpy() for f in fr])
    poses = np.stack([f["T_world_sensor"] for f in fr])
    swd, sw = orc.project_voxels(cfg["grid"], np.eye(4), depth, poses, cfg["sensor"], vox)
    assert np.array_equal(sw, W[keep].reshape(-1))
    obs = sw > 0
    assert obs.sum() > 1000
    assert np.allclose(swd[obs] / sw[obs], D[keep].reshape(-1)[obs], atol=1e-12)
