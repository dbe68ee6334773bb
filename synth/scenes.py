"""Analytic scenes, sensors and trajectories (seeded, synthetic).

Only input generation lives here: ray/primitive intersection of *ideal* sensor rays with
planes, yawed boxes and spheres, plus seeded noise.  The TSDF/ESDF method itself is
implemented twice elsewhere (oracle/ on the CPU, paper_2410_21149_b200/csrc on the GPU)
and neither half is imported by this module.

Conventions
-----------
* Poses are 4x4 fp64 numpy arrays, row-major, T_a_b maps b-coordinates into a.
* LiDAR sensor frame: x forward, y left, z up.  Organised output [rings*cols, 3] fp32,
  ring-major, NaN for "no return" (rays without a hit are not valid points).
* Pinhole camera frame: x right, y down, z forward.  Depth output [H, W] fp32 metres,
  0 for "no return".
* All random draws come from numpy PCG64 streams keyed by (seed, frame) so any subset of
  frames is reproducible on its own.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

F64 = torch.float64


# ----------------------------------------------------------------------------- scenes
@dataclass
class Scene:
    planes_n: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    planes_h: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    box_c: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    box_h: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))   # half extents
    box_yaw: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    sph_c: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    sph_r: np.ndarray = field(default_factory=lambda: np.zeros((0,)))


def _t(a, device):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), dtype=F64, device=device)


def raycast(scene: Scene, origin: np.ndarray, dirs: torch.Tensor, eps: float = 1e-9,
            chunk: int = 32) -> torch.Tensor:
    """Smallest positive ray parameter t with origin + t*dirs on a scene surface (inf if none).

    dirs: [N,3] fp64 tensor (need not be unit length).  Returns [N] fp64.
    """
    dev = dirs.device
    o = _t(origin, dev).reshape(1, 3)
    n = dirs.shape[0]
    best = torch.full((n,), math.inf, dtype=F64, device=dev)
    inf = torch.tensor(math.inf, dtype=F64, device=dev)

    def take(t):
        nonlocal best
        t = torch.where(t > eps, t, inf)
        best = torch.minimum(best, t.min(dim=1).values)

    # planes n.x = h
    for s in range(0, len(scene.planes_h), chunk):
        pn = _t(scene.planes_n[s:s + chunk], dev)              # [K,3]
        ph = _t(scene.planes_h[s:s + chunk], dev)              # [K]
        den = dirs @ pn.T                                      # [N,K]
        num = ph.reshape(1, -1) - (o @ pn.T)                   # [1,K]
        den = torch.where(den == 0, torch.full_like(den, 1e-300), den)
        take(num / den)
    # spheres
    for s in range(0, len(scene.sph_r), chunk):
        c = _t(scene.sph_c[s:s + chunk], dev)
        r = _t(scene.sph_r[s:s + chunk], dev)
        oc = (o - c)                                           # [K,3]
        a = (dirs * dirs).sum(1, keepdim=True)                 # [N,1]
        b = 2.0 * (dirs @ oc.T)                                # [N,K]
        cc = (oc * oc).sum(1) - r * r                          # [K]
        disc = b * b - 4.0 * a * cc.reshape(1, -1)
        sq = torch.sqrt(torch.clamp(disc, min=0.0))
        t1 = (-b - sq) / (2.0 * a)
        t2 = (-b + sq) / (2.0 * a)
        t = torch.where(t1 > eps, t1, t2)
        t = torch.where(disc >= 0, t, inf)
        take(t)
    # yawed boxes (slab test in the box frame)
    for s in range(0, len(scene.box_yaw), chunk):
        c = _t(scene.box_c[s:s + chunk], dev)
        h = _t(scene.box_h[s:s + chunk], dev)
        yaw = _t(scene.box_yaw[s:s + chunk], dev)
        cy, sy = torch.cos(yaw).reshape(1, -1), torch.sin(yaw).reshape(1, -1)
        oc = (o - c)                                           # [K,3]
        ox = cy * oc[:, 0].reshape(1, -1) + sy * oc[:, 1].reshape(1, -1)
        oy = -sy * oc[:, 0].reshape(1, -1) + cy * oc[:, 1].reshape(1, -1)
        oz = oc[:, 2].reshape(1, -1).expand_as(ox)
        dx = cy * dirs[:, 0:1] + sy * dirs[:, 1:2]
        dy = -sy * dirs[:, 0:1] + cy * dirs[:, 1:2]
        dz = dirs[:, 2:3].expand_as(dx)
        tmin = torch.full_like(dx, -math.inf)
        tmax = torch.full_like(dx, math.inf)
        for oa, da, ha in ((ox, dx, h[:, 0]), (oy, dy, h[:, 1]), (oz, dz, h[:, 2])):
            ha = ha.reshape(1, -1)
            da_safe = torch.where(da == 0, torch.full_like(da, 1e-300), da)
            ta = (-ha - oa) / da_safe
            tb = (ha - oa) / da_safe
            tmin = torch.maximum(tmin, torch.minimum(ta, tb))
            tmax = torch.minimum(tmax, torch.maximum(ta, tb))
        hit = tmax >= torch.clamp(tmin, min=eps)
        t = torch.where(tmin > eps, tmin, tmax)
        take(torch.where(hit, t, inf))
    return best


# ----------------------------------------------------------------------------- poses
def rot_zyx(yaw: float, pitch: float = 0.0, roll: float = 0.0) -> np.ndarray:
    cz, sz = math.cos(yaw), math.sin(yaw)
    cy, sy = math.cos(pitch), math.sin(pitch)
    cx, sx = math.cos(roll), math.sin(roll)
    rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1.0]])
    ry = np.array([[cy, 0, sy], [0, 1.0, 0], [-sy, 0, cy]])
    rx = np.array([[1.0, 0, 0], [0, cx, -sx], [0, sx, cx]])
    return rz @ ry @ rx


def pose(R: np.ndarray, t) -> np.ndarray:
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = np.asarray(t, dtype=np.float64)
    return T


# camera (x right, y down, z forward) looking along body +x of a z-up body frame
_BODY_FROM_CAM = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])


def camera_pose(position, yaw: float, pitch_down: float = 0.0, roll: float = 0.0) -> np.ndarray:
    """T_world_camera for a camera at `position` looking along yaw, pitched down by pitch_down."""
    R_wb = rot_zyx(yaw, pitch_down, roll)
    return pose(R_wb @ _BODY_FROM_CAM, position)


# ----------------------------------------------------------------------------- sensors
def lidar_directions(rings: int = 64, cols: int = 1024, fov_deg: float = 33.2) -> np.ndarray:
    """OS1-64-shaped unit directions [rings*cols, 3], ring-major (domain knowledge)."""
    half = math.radians(fov_deg / 2)
    el = np.linspace(-half, half, rings) if rings > 1 else np.zeros(1)
    az = 2.0 * math.pi * np.arange(cols) / cols
    E, A = np.meshgrid(el, az, indexing="ij")
    return np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)


def surface_color(hits_w: torch.Tensor) -> torch.Tensor:
    """Procedural surface texture: uint8 RGB [N,3] of world hit points (fp64 [N,3]; non-finite -> 0).
    Smooth in space, so neighbouring returns on a surface carry similar (not equal) colours."""
    x, y, z = hits_w[:, 0], hits_w[:, 1], hits_w[:, 2]
    c = torch.stack([128 + 127 * torch.sin(1.3 * x) * torch.cos(0.7 * y),
                     128 + 127 * torch.sin(0.9 * z + 0.5 * x),
                     128 + 127 * torch.cos(0.4 * (x + y + z))], -1)
    c = torch.where(torch.isfinite(c), c, torch.zeros_like(c))
    return torch.clamp(torch.floor(c), 0, 255).to(torch.uint8)


def lidar_scan(scene: Scene, T_ws: np.ndarray, dirs_s: np.ndarray, r_max: float, sigma: float,
               rng: np.random.Generator, device="cpu", color: bool = False):
    """Organised LiDAR scan in the sensor frame, fp32 [N,3]; NaN where there is no return.
    color=True also returns the uint8 [N,3] surface colour of each return (0 where none)."""
    d_s = _t(dirs_s, device)
    R = _t(T_ws[:3, :3], device)
    t = raycast(scene, T_ws[:3, 3], d_s @ R.T)
    if color:
        rgb = surface_color(_t(T_ws[:3, 3], device) + (d_s @ R.T) * t.reshape(-1, 1))
        return lidar_scan(scene, T_ws, dirs_s, r_max, sigma, rng, device), rgb
    noise = _t(rng.normal(0.0, sigma, size=len(dirs_s)), device) if sigma > 0 else 0.0
    ok = t <= r_max
    r = t + noise
    pts = d_s * r.reshape(-1, 1)
    pts = torch.where(ok.reshape(-1, 1), pts, torch.full_like(pts, math.nan))
    return pts.to(torch.float32)


def pinhole_rays(width: int, height: int, fx: float, fy: float, cx: float, cy: float) -> np.ndarray:
    """Camera-frame ray directions with unit z component, [H*W,3] (integer pixel indices)."""
    v, u = np.meshgrid(np.arange(height, dtype=np.float64), np.arange(width, dtype=np.float64), indexing="ij")
    return np.stack([(u - cx) / fx, (v - cy) / fy, np.ones_like(u)], -1).reshape(-1, 3)


def pinhole_depth(scene: Scene, T_wc: np.ndarray, cam: dict, r_max: float, noise_k: float,
                  rng: np.random.Generator, device="cpu", color: bool = False):
    """Depth image fp32 [H,W] (z along the optical axis); 0 where there is no return.
    color=True also returns the uint8 [H*W,3] surface colour per pixel (0 where no return)."""
    d_c = _t(pinhole_rays(cam["width"], cam["height"], cam["fx"], cam["fy"], cam["cx"], cam["cy"]), device)
    R = _t(T_wc[:3, :3], device)
    z = raycast(scene, T_wc[:3, 3], d_c @ R.T)       # unit-z rays: parameter == depth
    if color:
        rgb = surface_color(_t(T_wc[:3, 3], device) + (d_c @ R.T) * z.reshape(-1, 1))
        return pinhole_depth(scene, T_wc, cam, r_max, noise_k, rng, device), rgb
    ok = (z * torch.linalg.norm(d_c, dim=1)) <= r_max
    if noise_k > 0:
        z = z + _t(rng.normal(0.0, 1.0, size=z.shape[0]), device) * noise_k * z * z
    z = torch.where(ok & torch.isfinite(z), z, torch.zeros_like(z))
    return z.reshape(cam["height"], cam["width"]).to(torch.float32)


# ----------------------------------------------------------------------------- configs
def _grid(voxel_size, truncation, max_blocks, weighting=0, carve=1, site_threshold=None):
    return dict(voxel_size=voxel_size, block_side=8, truncation=truncation, weighting=weighting,
                weight_range_floor=0.1, carve=carve,
                site_threshold=voxel_size if site_threshold is None else site_threshold,
                max_blocks=max_blocks, esdf_max_distance=2.0)


def _tiny_scene():
    return Scene(planes_n=np.array([[0.0, 0.0, 1.0]]), planes_h=np.array([0.0]),
                 sph_c=np.array([[2.0, 0.0, 0.5]]), sph_r=np.array([0.5]))


def _city_scene(seed: int, half: float = 60.0, n_boxes: int = 50, n_sph: int = 200,
                corridor=((-25.0, 25.0), (-6.0, 6.0))) -> Scene:
    rng = np.random.Generator(np.random.PCG64(seed))
    bc, bh, by = [], [], []
    while len(bc) < n_boxes:
        c = rng.uniform(-half, half, 2)
        hx, hy = rng.uniform(2.5, 10.0, 2)
        hz = rng.uniform(2.5, 10.0)
        rr = math.hypot(hx, hy)
        if corridor[0][0] - rr < c[0] < corridor[0][1] + rr and corridor[1][0] - rr < c[1] < corridor[1][1] + rr:
            continue
        bc.append([c[0], c[1], hz]); bh.append([hx, hy, hz]); by.append(rng.uniform(0, math.pi))
    sc, sr = [], []
    while len(sc) < n_sph:
        c = rng.uniform(-half, half, 2)
        r = rng.uniform(0.3, 2.0)
        if corridor[0][0] - 2 < c[0] < corridor[0][1] + 2 and abs(c[1]) < 3.5:
            continue
        sc.append([c[0], c[1], 0.5 * r]); sr.append(r)
    return Scene(planes_n=np.array([[0.0, 0.0, 1.0]]), planes_h=np.array([0.0]),
                 box_c=np.array(bc), box_h=np.array(bh), box_yaw=np.array(by),
                 sph_c=np.array(sc), sph_r=np.array(sr))


def _room_scene(seed: int) -> Scene:
    rng = np.random.Generator(np.random.PCG64(seed))
    # room 10 x 8 x 3 m (sensor inside: the far slab face is hit) + 20 furniture boxes
    bc = [[0.0, 0.0, 1.5]]; bh = [[5.0, 4.0, 1.5]]; by = [0.0]
    while len(bc) < 21:
        c = rng.uniform([-4.3, -3.3], [4.3, 3.3])
        if abs(c[0]) < 3.6 and abs(c[1]) < 2.6 and math.hypot(c[0] / 3.0, c[1] / 2.0) > 0.55 \
                and math.hypot(c[0] / 3.0, c[1] / 2.0) < 1.45:
            continue                                   # keep the camera loop free
        hx, hy, hz = rng.uniform(0.15, 0.75, 3)
        bc.append([c[0], c[1], hz]); bh.append([hx, hy, hz]); by.append(rng.uniform(0, math.pi))
    return Scene(box_c=np.array(bc), box_h=np.array(bh), box_yaw=np.array(by))


def _mav_scene(seed: int) -> Scene:
    """200 x 120 m disaster site: ground, rubble pile, scattered debris, one enterable building."""
    s = _city_scene(seed, half=60.0, n_boxes=25, n_sph=150, corridor=((-1e9, -1e9), (0, 0)))
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    # rubble pile (foreground of Fig. 1)
    pile_c = rng.normal([40.0, 25.0], 6.0, size=(250, 2))
    pile_r = rng.uniform(0.4, 2.5, 250)
    sph_c = np.concatenate([s.sph_c, np.column_stack([pile_c, pile_r * 0.3])])
    sph_r = np.concatenate([s.sph_r, pile_r])
    # building 16 x 24 x 8 m centred at (-82, 0) with 6 m door gaps in the y faces: the flight path
    # passes through it (indoor-outdoor transitions)
    walls_c, walls_h = [], []
    cx0, cy0, hx, hy, hz, t = -82.0, 0.0, 8.0, 12.0, 4.0, 0.2
    for side in (-1, 1):
        walls_c.append([cx0 + side * hx, cy0, hz]); walls_h.append([t, hy, hz])          # long walls
        for part in (-1, 1):                                                          # y walls with a 6 m door
            walls_c.append([cx0 + part * (hx + 3.0) / 2, cy0 + side * hy, hz])
            walls_h.append([(hx - 3.0) / 2, t, hz])
    walls_c.append([cx0, cy0, 2 * hz]); walls_h.append([hx, hy, t])                    # roof
    box_c = np.concatenate([s.box_c, np.array(walls_c)])
    box_h = np.concatenate([s.box_h, np.array(walls_h)])
    box_yaw = np.concatenate([s.box_yaw, np.zeros(len(walls_c))])
    return Scene(planes_n=s.planes_n, planes_h=s.planes_h, box_c=box_c, box_h=box_h, box_yaw=box_yaw,
                 sph_c=sph_c, sph_r=sph_r)


CONFIGS = ("tiny", "lidar", "rgbd", "mav")


def make_config(name: str, frames=None, device="cpu", seed=None, lidar_cols: int = 1024, color: bool = False):
    """Build one BASELINE.json config as posed frames.

    Returns dict(name, grid, sensor, submaps=[dict(T_world_submap, frames=[idx...])],
    frames=[dict(data=fp32 tensor, T_world_sensor=4x4)]).  `frames` selects a subset of
    frame indices (the rest are not generated).  color=True adds per-point surface colour
    (uint8 [n,3], frame["rgb"]) for TSDF + Color.
    """
    if name == "tiny":                                   # BJ.configs[0]
        seed = 0 if seed is None else seed
        scene = _tiny_scene()
        cam = dict(kind=1, width=64, height=48, fx=40.0, fy=40.0, cx=31.5, cy=23.5, min_range=0.1, max_range=5.0)
        n_frames = 10
        poses = [camera_pose([0.0, -0.45 + 0.1 * k, 1.0], 0.0, math.radians(15.0)) for k in range(n_frames)]
        grid = _grid(0.1, 0.3, 1 << 13)
        gen = lambda k, T, rng: pinhole_depth(scene, T, cam, cam["max_range"], 0.0, rng, device, color)  # noqa: E731
        submaps = [dict(T_world_submap=np.eye(4), frames=list(range(n_frames)))]
        sensor = cam
    elif name in ("lidar", "mav"):                       # BJ.configs[1], [3]
        seed = (1 if name == "lidar" else 3) if seed is None else seed
        scene = _city_scene(seed) if name == "lidar" else _mav_scene(seed)
        sensor = dict(kind=2, width=lidar_cols, height=64, fx=0.0, fy=0.0, cx=0.0, cy=0.0,
                      min_range=0.5, max_range=100.0)
        dirs = lidar_directions(64, lidar_cols)
        rng0 = np.random.Generator(np.random.PCG64(seed + 77))
        if name == "lidar":
            n_frames = 200
            poses = []
            for k in range(n_frames):
                rp = rng0.uniform(-math.radians(2), math.radians(2), 2)
                poses.append(pose(rot_zyx(math.radians(0.5 * k), rp[0], rp[1]), [-20.0 + 0.2 * k, 0.0, 3.0]))
            submaps = [dict(T_world_submap=pose(rot_zyx(math.radians(10.0)), [-20.0, 0.0, 0.0]),
                            frames=list(range(n_frames)))]
            grid = _grid(0.2, 0.6, 1 << 19)
        else:
            n_frames = 2000
            poses = []
            # ~400 m elliptic loop (a = 82 m, b = 41 m) at 2-6 m altitude through the building
            for k in range(n_frames):
                th = 2 * math.pi * k / n_frames
                x, y = 82.0 * math.cos(th), 41.0 * math.sin(th)
                z = 4.0 + 2.0 * math.sin(4 * th)
                if abs(x + 82.0) < 10.0 and abs(y) < 14.0:   # inside the building: fly low
                    z = 2.0
                yaw = math.atan2(41.0 * math.cos(th), -82.0 * math.sin(th))
                rp = rng0.uniform(-math.radians(2), math.radians(2), 2)
                poses.append(pose(rot_zyx(yaw, rp[0], rp[1]), [x, y, z]))
            submaps = []
            for m in range(40):                          # 40 submaps x 50 contiguous scans
                k0 = 50 * m
                submaps.append(dict(T_world_submap=pose(np.eye(3), poses[k0][:3, 3] * np.array([1, 1, 0])),
                                    frames=list(range(k0, k0 + 50))))
            grid = _grid(0.2, 0.6, 1 << 19)
        gen = lambda k, T, rng: lidar_scan(scene, T, dirs, sensor["max_range"], 0.02, rng, device, color)  # noqa: E731
    elif name == "rgbd":                                 # BJ.configs[2]
        seed = 2 if seed is None else seed
        scene = _room_scene(seed)
        sensor = dict(kind=1, width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5,
                      min_range=0.1, max_range=5.0)
        n_frames = 1000
        poses = []
        for k in range(n_frames):
            a = 2 * math.pi * k / n_frames
            p = [3.0 * math.cos(a), 2.0 * math.sin(a), 1.5 + 0.3 * math.sin(5 * a)]
            yaw = a + math.pi / 2 + 0.6 * math.sin(3 * a)   # tangent, swinging towards the walls
            poses.append(camera_pose(p, yaw, math.radians(10.0 + 8.0 * math.sin(2 * a))))
        submaps = [dict(T_world_submap=pose(np.eye(3), [0.0, 0.0, 0.0]), frames=list(range(100 * m, 100 * m + 100)))
                   for m in range(10)]
        grid = _grid(0.05, 0.15, 1 << 16)
        gen = lambda k, T, rng: pinhole_depth(scene, T, sensor, sensor["max_range"], 0.0012, rng, device, color)  # noqa: E731
    else:
        raise ValueError(f"unknown config {name!r}")

    idx = range(n_frames) if frames is None else frames
    out_frames = {}
    for k in idx:
        rng = np.random.Generator(np.random.PCG64([seed, int(k)]))
        g = gen(k, poses[k], rng)
        if color:
            out_frames[int(k)] = dict(data=g[0], rgb=g[1], T_world_sensor=poses[k])
        else:
            out_frames[int(k)] = dict(data=g, T_world_sensor=poses[k])
    return dict(name=name, grid=grid, sensor=sensor, submaps=submaps, frames=out_frames,
                poses=poses, n_frames=n_frames, seed=seed)


# ----------------------------------------------------------------------------- ESDF stress (configs[4])
def esdf_stress_scene(seed: int = 4, extent=(40.0, 40.0, 10.0), n_boxes: int = 60, n_spheres: int = 40):
    """~100 analytic boxes / spheres on a ground plane inside a 40 x 40 x 10 m volume."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ex, ey, ez = extent
    bc = np.column_stack([rng.uniform(1, ex - 1, n_boxes), rng.uniform(1, ey - 1, n_boxes), np.zeros(n_boxes)])
    bh = np.column_stack([rng.uniform(0.2, 2.5, n_boxes), rng.uniform(0.2, 2.5, n_boxes), rng.uniform(0.3, 4.0, n_boxes)])
    bc[:, 2] = bh[:, 2]
    sc = np.column_stack([rng.uniform(1, ex - 1, n_spheres), rng.uniform(1, ey - 1, n_spheres),
                          rng.uniform(0.3, max(0.6, ez - 0.5), n_spheres)])
    sr = rng.uniform(0.2, 1.5, n_spheres)
    return dict(box_c=bc, box_h=bh, sph_c=sc, sph_r=sr, extent=extent)


def analytic_sdf(scene: dict, pts: torch.Tensor) -> torch.Tensor:
    """Signed distance (m, negative inside) of the union of ground (z = 0), boxes and spheres at pts [N,3]."""
    dev = pts.device
    sdf = pts[:, 2].clone()                                               # ground plane z = 0
    for c, h in zip(scene["box_c"], scene["box_h"]):
        q = (pts - torch.tensor(c, dtype=pts.dtype, device=dev)).abs() - torch.tensor(h, dtype=pts.dtype, device=dev)
        d = q.clamp(min=0).norm(dim=1) + q.max(dim=1).values.clamp(max=0)
        sdf = torch.minimum(sdf, d)
    for c, r in zip(scene["sph_c"], scene["sph_r"]):
        d = (pts - torch.tensor(c, dtype=pts.dtype, device=dev)).norm(dim=1) - float(r)
        sdf = torch.minimum(sdf, d)
    return sdf


def esdf_stress_blocks(voxel_size: float = 0.02, truncation: float = 0.06, extent=(40.0, 40.0, 10.0),
                       z0: float = -0.5, device="cuda", chunk_blocks: int = 1 << 15, seed: int = 4,
                       n_boxes: int = 60, n_spheres: int = 40):
    """Yield (bxyz int32 [n,3], D fp32 [n,512], W fp32 [n,512]) chunks of a fully observed TSDF
    D = clamp(analytic sdf, +-tau), W = 1 over the volume (BASELINE.json configs[4]).  Block (bx,by,bz)
    covers voxels 8*b .. 8*b+7; voxel centres at (v + 1/2) s in the submap frame, z offset z0."""
    scene = esdf_stress_scene(seed, extent, n_boxes, n_spheres)
    nbx, nby, nbz = (int(round(e / voxel_size)) // 8 for e in extent)
    bz0 = int(np.floor(z0 / voxel_size / 8))
    l = torch.arange(512, device=device)
    loc = torch.stack([l % 8, (l // 8) % 8, l // 64], 1).to(torch.float32)
    total = nbx * nby * nbz
    for s0 in range(0, total, chunk_blocks):
        ids = torch.arange(s0, min(total, s0 + chunk_blocks), device=device)
        b = torch.stack([ids % nbx, (ids // nbx) % nby, ids // (nbx * nby) + bz0], 1).to(torch.int32)
        v = b.to(torch.float32)[:, None, :] * 8 + loc[None]
        pts = ((v + 0.5) * voxel_size).reshape(-1, 3)
        sdf = analytic_sdf(scene, pts).reshape(-1, 512)
        D = sdf.clamp(-truncation, truncation).contiguous()
        W = torch.ones_like(D)
        yield b.contiguous(), D, W
