"""Pins of the oracle's TSDF.

References: the S:L272-274 worked example, the single-ray closed-form ramp, same frame
twice, permutation invariance, clamping, the analytic parallel-ray
plane (exact closed form), the oblique-plane and hollow-sphere error bounds (SURVEY §8c pins),
exact rigid-motion equivariance of the pose composition (O1), and the depth->point formula (O2)
checked against an analytic plane.
"""
import math

import numpy as np
import pytest

import synth


def _one_ray(orc, o, p_c, grid, weighting=0):
    g = dict(grid)
    g["weighting"] = weighting
    sm = orc.OracleSubmap(g)
    T = np.eye(4)
    T[:3, 3] = o
    sensor = dict(kind=0, min_range=0.0, max_range=1e9)
    sm.integrate(np.asarray([p_c], np.float32), T, sensor)
    return sm


def _voxel_table(sm):
    b, D, W = sm.export()
    out = {}
    for i in range(b.shape[0]):
        for l in range(512):
            if W[i, l] > 0:
                v = (8 * b[i, 0] + l % 8, 8 * b[i, 1] + (l // 8) % 8, 8 * b[i, 2] + l // 64)
                out[v] = (D[i, l], W[i, l])
    return out


GRID = dict(voxel_size=0.05, truncation=0.15, weighting=0, weight_range_floor=0.1, carve=1,
            site_threshold=0.05, max_blocks=1 << 12)


def test_paper_example_sdf_and_weight(orc):
    # voxel centre at the surface -> sdf 0; voxel 0.05 m in front on a 2 m ray with
    # inverse-square weighting -> sdf +0.05, weight 1/2^2 = 0.25
    o = np.array([0.025, 0.025, 0.025])
    sm = _one_ray(orc, o, [2.0, 0.0, 0.0], GRID, weighting=1)
    t = _voxel_table(sm)
    d40, w40 = t[(40, 0, 0)]          # centre 2.025 == p
    d39, w39 = t[(39, 0, 0)]          # centre 1.975, 0.05 m in front
    assert abs(d40) < 1e-12 and abs(d39 - 0.05) < 1e-12
    assert w40 == pytest.approx(0.25, abs=1e-15) and w39 == pytest.approx(0.25, abs=1e-15)


def test_single_ray_linear_ramp(orc):
    # one point straight ahead, constant weights -> clamped linear ramp, all weights 1;
    # carving from the optical centre to tau behind the point
    o = np.array([0.025, 0.025, 0.025])
    sm = _one_ray(orc, o, [1.0, 0.0, 0.0], GRID)
    t = _voxel_table(sm)
    xs = sorted(k[0] for k in t)
    assert xs == list(range(0, 24))   # 0.025 -> 1.025 + 0.15 = 1.175 -> voxels 0..23
    for (x, y, z), (d, w) in t.items():
        c = (x + 0.5) * 0.05
        assert w == 1.0
        assert d == pytest.approx(min(max(1.025 - c, -0.15), 0.15), abs=1e-12)
    assert max(abs(d) for d, _ in t.values()) <= 0.15


def test_same_frame_twice_and_permutation(orc):
    cfg = synth.make_config("tiny", frames=[0])
    fr = cfg["frames"][0]
    a = orc.OracleSubmap(cfg["grid"])
    a.integrate(fr["data"].numpy(), fr["T_world_sensor"], cfg["sensor"])
    b1, D1, W1 = a.export()
    a.integrate(fr["data"].numpy(), fr["T_world_sensor"], cfg["sensor"])
    b2, D2, W2 = a.export()
    assert (b1 == b2).all()                        # same block set
    assert np.array_equal(W2, 2 * W1)              # weights doubled exactly
    assert np.allclose(D2, D1, atol=1e-12)         # distances unchanged
    assert np.abs(D1).max() <= cfg["grid"]["truncation"] * (1 + 1e-12)   # S:L303 clamp (mean of clamped)
    # permuting the points of a cloud does not change the state
    from oracle import OracleSubmap
    cfgl = synth.make_config("lidar", frames=[0], lidar_cols=128)
    pts = cfgl["frames"][0]["data"].numpy()
    perm = np.random.default_rng(0).permutation(pts.shape[0])
    s1 = OracleSubmap(cfgl["grid"], cfgl["submaps"][0]["T_world_submap"])
    s2 = OracleSubmap(cfgl["grid"], cfgl["submaps"][0]["T_world_submap"])
    st1 = s1.integrate(pts, cfgl["frames"][0]["T_world_sensor"], cfgl["sensor"])
    st2 = s2.integrate(pts[perm], cfgl["frames"][0]["T_world_sensor"], cfgl["sensor"])
    assert st1 == st2
    e1, e2 = s1.export(), s2.export()
    assert (e1[0] == e2[0]).all() and np.array_equal(e1[2], e2[2])
    assert np.allclose(e1[1], e2[1], atol=1e-12)


def test_weight_monotone(orc):
    cfg = synth.make_config("tiny", frames=[0, 1, 2])
    s = orc.OracleSubmap(cfg["grid"])
    prev = {}
    for k in (0, 1, 2):
        fr = cfg["frames"][k]
        s.integrate(fr["data"].numpy(), fr["T_world_sensor"], cfg["sensor"])
        t = _voxel_table(s)
        for v, (_, w) in prev.items():
            assert t[v][1] >= w
        prev = t


def test_parallel_ray_plane_closed_form(orc):
    # Every frame holds one point on the plane z = h seen from straight above, so every ray is
    # normal to the plane and D(v) = clamp(c_z - h, -tau, tau) exactly (SURVEY §8c pins).
    rng = np.random.default_rng(3)
    g = dict(GRID, voxel_size=0.1, truncation=0.3)
    h = 0.4375
    s = orc.OracleSubmap(g)
    sensor = dict(kind=0, min_range=0.0, max_range=1e9)
    for _ in range(300):
        x, y = rng.uniform(-3, 3, 2)
        H = rng.integers(256, 2048) / 512.0            # exact in fp32
        T = np.eye(4)
        T[:3, 3] = [x, y, h + H]
        s.integrate(np.array([[0.0, 0.0, -H]], np.float32), T, sensor)
    t = _voxel_table(s)
    assert len(t) > 1000
    for (vx, vy, vz), (d, w) in t.items():
        c = (vz + 0.5) * 0.1
        assert d == pytest.approx(min(max(c - h, -0.3), 0.3), abs=1e-9)


def _plane_scene_lidar(orc, theta_max_deg):
    """Sensor above plane z=0 with rays of incidence <= theta_max (downward cone)."""
    rng = np.random.default_rng(11)
    g = dict(GRID, voxel_size=0.1, truncation=0.3)
    s = orc.OracleSubmap(g)
    sensor = dict(kind=0, min_range=0.0, max_range=1e9)
    th = math.radians(theta_max_deg)
    for k in range(6):
        Hs = 2.0 + 0.37 * k
        n = 3000
        ct = rng.uniform(math.cos(th), 1.0, n)
        st = np.sqrt(1 - ct * ct)
        ph = rng.uniform(0, 2 * math.pi, n)
        u = np.stack([st * np.cos(ph), st * np.sin(ph), -ct], 1)
        pts = u * (Hs / ct)[:, None]                   # on z = 0 (up to fp32 rounding)
        T = np.eye(4)
        T[:3, 3] = [0.3 * k, -0.2 * k, Hs]
        s.integrate(pts.astype(np.float32), T, sensor)
    return s, th, g


def test_oblique_plane_bound(orc):
    # |D - clamp(delta)| <= |delta| (sec th - 1) + (s sqrt3/2) tan th, per ray and so for the mean
    s, th, g = _plane_scene_lidar(orc, 30.0)
    vs = g["voxel_size"]
    t = _voxel_table(s)
    bad = 0
    for (vx, vy, vz), (d, w) in t.items():
        delta = (vz + 0.5) * vs
        bound = abs(delta) * (1 / math.cos(th) - 1) + vs * math.sqrt(3) / 2 * math.tan(th)
        if abs(d - min(max(delta, -0.3), 0.3)) > bound + 1e-5:
            bad += 1
    assert bad == 0


def test_hollow_sphere_bound(orc):
    # Sensor at the centre of a hollow sphere: rays radial; 0 <= D - clamp(delta) <= 3s^2/(8(|c-o| - s sqrt3/2))
    rng = np.random.default_rng(5)
    vs, tau, R = 0.1, 0.3, 2.0
    g = dict(GRID, voxel_size=vs, truncation=tau)
    s = orc.OracleSubmap(g)
    o = np.array([0.013, -0.021, 0.007])
    u = rng.normal(size=(20000, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    T = np.eye(4)
    T[:3, 3] = o
    s.integrate((u * R).astype(np.float32), T, dict(kind=0, min_range=0.0, max_range=1e9))
    t = _voxel_table(s)
    n = 0
    for v, (d, w) in t.items():
        c = (np.array(v) + 0.5) * vs
        r = np.linalg.norm(c - o)
        if r < 0.5:
            continue
        delta = R - r
        bound = 3 * vs * vs / (8 * (r - vs * math.sqrt(3) / 2))
        diff = d - min(max(delta, -tau), tau)
        assert -2e-6 <= diff <= bound + 2e-6, (v, diff, bound)
        n += 1
    assert n > 5000


def test_pose_composition_equivariance(orc):
    # O1: moving both the submap and the sensor by the same rigid motion leaves the submap-frame
    # TSDF unchanged.  A 90-degree yaw and a translation by whole blocks are exact in fp64.
    cfg = synth.make_config("lidar", frames=[0], lidar_cols=128)
    fr = cfg["frames"][0]
    g = dict(cfg["grid"], voxel_size=0.25, truncation=0.75)
    M = np.array([[0.0, -1.0, 0.0, 4.0], [1.0, 0.0, 0.0, -6.0], [0.0, 0.0, 1.0, 2.0], [0, 0, 0, 1.0]])
    T_ws = np.eye(4)
    T_ws[:3, 3] = [-8.0, 2.0, 0.0]
    T_wc = fr["T_world_sensor"].copy()
    T_wc[:3, 3] = np.round(T_wc[:3, 3] * 64) / 64            # dyadic sensor position
    T_wc[:3, :3] = np.eye(3)
    a = orc.OracleSubmap(g, T_ws)
    a.integrate(fr["data"].numpy(), T_wc, cfg["sensor"])
    b = orc.OracleSubmap(g, M @ T_ws)
    b.integrate(fr["data"].numpy(), M @ T_wc, cfg["sensor"])
    ea, eb = a.export(), b.export()
    assert (ea[0] == eb[0]).all()
    assert np.array_equal(ea[2], eb[2])
    assert np.allclose(ea[1], eb[1], atol=1e-12)


def test_depth_backprojection_plane(orc):
    # O2: a pinhole depth image of the plane z_cam = 2 (every pixel depth 2) back-projects to points
    # on that plane, so with the camera looking straight down at ground z = 0 from 2 m, the observed
    # surface voxels obey the oblique-plane bound for the image's maximum incidence angle.
    W_, H_ = 16, 12
    sensor = dict(kind=1, width=W_, height=H_, fx=20.0, fy=20.0, cx=7.5, cy=5.5, min_range=0.0, max_range=10.0)
    depth = np.full((H_, W_), 2.0, np.float32)
    T = synth.camera_pose([0.0, 0.0, 2.0], 0.0, math.radians(90.0))
    g = dict(GRID, voxel_size=0.1, truncation=0.3)
    s = orc.OracleSubmap(g)
    st = s.integrate(depth, T, sensor)
    assert st["rays_used"] == W_ * H_
    th = math.atan(math.hypot(7.5 / 20.0, 5.5 / 20.0))
    t = _voxel_table(s)
    for (vx, vy, vz), (d, w) in t.items():
        delta = (vz + 0.5) * 0.1
        bound = abs(delta) * (1 / math.cos(th) - 1) + 0.1 * math.sqrt(3) / 2 * math.tan(th)
        assert abs(d - min(max(delta, -0.3), 0.3)) <= bound + 1e-5
    # (the pixel -> point mapping itself is pinned exactly, pixel by pixel, in
    # test_depth_backprojection_exact_per_pixel below)
    b, D, Wt = s.export()
    assert (Wt > 0).sum() == len(t)


def test_invalid_and_range_counting(orc):
    s = orc.OracleSubmap(GRID)
    pts = np.array([[1, 0, 0], [np.nan, 0, 0], [0, np.inf, 0], [0.01, 0, 0], [50, 0, 0]], np.float32)
    st = s.integrate(pts, np.eye(4), dict(kind=0, min_range=0.1, max_range=10.0))
    assert st["rays_in"] == 5 and st["rays_used"] == 1
    assert st["skipped_invalid"] == 2 and st["skipped_range"] == 2
    st = s.integrate(np.zeros((0, 3), np.float32), np.eye(4), dict(kind=0, min_range=0.1, max_range=10.0))
    assert st["rays_in"] == 0 and st["voxel_updates"] == 0   # S:L283 empty frame is a no-op


def test_depth_backprojection_exact_per_pixel(orc):
    """O2 pinned pixel by pixel: pixel (u, v) = (i % W, i // W) of a W x H depth image
    with depth z back-projects to p_c = (z (u - cx) / fx, z (v - cy) / fy, z), integer pixel indices, no
    +1/2.  W != H, cx != (W-1)/2, cy != (H-1)/2 and a distinct dyadic depth per pixel, so every input is
    exact in fp32 and the expected point is an exact rational; only one pixel is valid per frame, so the
    observed voxels are exactly that ray's traversal (pinned separately, test_oracle_traversal.py) and
    D on them is the closed-form clamped sdf (p - c_v).u of the exact point.  A u/v swap, a transposed
    index (i % H), a +1/2 pixel centre or swapped intrinsics moves the point by >= 1 voxel and fails."""
    from fractions import Fraction as Fr
    W_, H_ = 5, 3
    fx, fy, cx, cy = 4.0, 2.0, 1.25, 0.5            # dyadic: fp32 arithmetic below is exact
    sensor = dict(kind=1, width=W_, height=H_, fx=fx, fy=fy, cx=cx, cy=cy, min_range=0.0, max_range=100.0)
    g = dict(GRID, voxel_size=0.05, truncation=0.1)
    s, tau = g["voxel_size"], g["truncation"]
    for i in range(W_ * H_):
        u, v = i % W_, i // W_
        z = 1.0 + i / 8.0                              # distinct per pixel, dyadic
        depth = np.zeros((H_, W_), np.float32)
        depth[v, u] = z
        p = [Fr(z) * (Fr(u) - Fr(cx)) / Fr(fx), Fr(z) * (Fr(v) - Fr(cy)) / Fr(fy), Fr(z)]
        pf = np.array([float(c) for c in p])
        assert all(Fr(float(c)) == c for c in p)       # the expected point is exact in fp64
        sm = orc.OracleSubmap(g)
        st = sm.integrate(depth, np.eye(4), sensor)
        assert st["rays_used"] == 1 and st["skipped_invalid"] == W_ * H_ - 1
        expect = orc.ray_voxels(np.zeros(3), pf, s, tau, 1)
        got = _voxel_table(sm)
        assert set(got) == set(map(tuple, expect.tolist())), (u, v)
        assert st["voxel_updates"] == expect.shape[0]
        L = float(np.sqrt(pf @ pf))
        assert abs(L - math.sqrt(float(sum(c * c for c in p)))) == 0.0
        uhat = pf / L
        for vox, (d, w) in got.items():
            c = (np.array(vox, np.float64) + 0.5) * s
            assert w == 1.0
            assert abs(d - min(max(float((pf - c) @ uhat), -tau), tau)) <= 1e-12
        # the ray ends tau behind the exact point: its last voxel holds e = p + tau u
        e = pf + tau * uhat
        assert tuple(expect[-1].tolist()) == tuple(int(np.floor(c / s)) for c in e)
