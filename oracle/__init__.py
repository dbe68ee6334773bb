"""ctypes front-end of the CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg are the only callers.  The product package never imports this module.
The oracle follows SURVEY.md §8c O1-O13 (and DESIGN.md "Readings"); see oracle.cpp for the
per-function citations.  Parity pinned: every function here is pinned by tests/test_oracle_*.py
(closed forms, brute force, scipy, paper examples) — no function is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (no FMA contraction: fp64 evaluated exactly as written)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Grid(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("truncation", C.c_double), ("weighting", C.c_int32),
                ("weight_range_floor", C.c_double), ("carve", C.c_int32), ("site_threshold", C.c_double)]


class Sensor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("min_range", C.c_float), ("max_range", C.c_float)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("rays_in", "rays_used", "skipped_invalid", "skipped_range",
                                         "skipped_domain", "voxel_updates", "new_blocks", "total_blocks")]

    def asdict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            P = C.c_void_p
            L.orc_new.restype = P
            L.orc_new.argtypes = [C.POINTER(Grid), P]
            L.orc_free.argtypes = [P]
            L.orc_integrate.restype = C.c_int32
            L.orc_integrate.argtypes = [P, P, C.c_int64, P, C.POINTER(Sensor), C.POINTER(Stats)]
            L.orc_integrate_color.restype = C.c_int32
            L.orc_integrate_color.argtypes = [P, P, P, C.c_int64, P, C.POINTER(Sensor), C.POINTER(Stats)]
            L.orc_export_color.argtypes = [P, P, P]
            L.orc_project_voxels.argtypes = [C.POINTER(Grid), P, P, C.c_int32, P, C.POINTER(Sensor), P, C.c_int64, P, P]
            L.orc_integrate_projective.restype = C.c_int32
            L.orc_integrate_projective.argtypes = [P, P, C.c_int64, P, C.POINTER(Sensor), C.POINTER(Stats)]
            L.orc_num_blocks.restype = C.c_int64
            L.orc_num_blocks.argtypes = [P]
            L.orc_export.argtypes = [P, P, P, P]
            L.orc_ray_voxels.restype = C.c_int64
            L.orc_ray_voxels.argtypes = [P, P, C.c_double, C.c_double, C.c_int32, P, C.c_int64]
            L.orc_esdf.restype = C.c_int32
            L.orc_esdf.argtypes = [P, P, P, C.c_int64, C.c_double, C.c_double, C.c_int32, P, P]
            L.orc_esdf_capped.restype = C.c_int32
            L.orc_esdf_capped.argtypes = [P, P, P, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int32, P]
            L.orc_esdf_sample.restype = C.c_int32
            L.orc_esdf_sample.argtypes = [P, P, P, C.c_int64, C.c_double, P, C.c_int64, P]
            L.orc_query.restype = C.c_int32
            L.orc_query.argtypes = [P, P, C.c_int64, C.c_double, P, P, C.c_int64, P, P, P]
            L.orc_sample_surface.restype = C.c_int32
            L.orc_sample_surface.argtypes = [P, P, P, C.c_int64, C.c_double, C.c_double, P, P, C.c_int64, P, P, P]
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def grid_struct(grid: dict) -> Grid:
    return Grid(float(grid["voxel_size"]), float(grid["truncation"]), int(grid.get("weighting", 0)),
                float(grid.get("weight_range_floor", 0.1)), int(grid.get("carve", 1)),
                float(grid.get("site_threshold", grid["voxel_size"])))


def sensor_struct(sensor: dict) -> Sensor:
    return Sensor(int(sensor["kind"]), int(sensor.get("width", 0)), int(sensor.get("height", 0)),
                  float(sensor.get("fx", 0)), float(sensor.get("fy", 0)), float(sensor.get("cx", 0)),
                  float(sensor.get("cy", 0)), float(sensor.get("min_range", 0.0)),
                  float(sensor.get("max_range", 3.0e38)))


class OracleSubmap:
    """One submap's TSDF as plain fp64 sums (O7-O8)."""

    def __init__(self, grid: dict, T_world_submap=None):
        self.grid = dict(grid)
        self._g = grid_struct(grid)
        T = np.ascontiguousarray(np.eye(4) if T_world_submap is None else T_world_submap, dtype=np.float64)
        self.T_ws = T
        self._h = lib().orc_new(C.byref(self._g), _p(T))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.orc_free(h)
            except Exception:
                pass
            self._h = None

    def integrate(self, data, T_world_sensor, sensor: dict) -> dict:
        d = np.ascontiguousarray(np.asarray(data, dtype=np.float32))
        n = d.size if sensor["kind"] == 1 else d.size // 3
        T = np.ascontiguousarray(T_world_sensor, dtype=np.float64)
        st = Stats()
        sm = sensor_struct(sensor)
        rc = lib().orc_integrate(self._h, _p(d), n, _p(T), C.byref(sm), C.byref(st))
        assert rc == 0
        return st.asdict()

    def integrate_projective(self, depth, T_world_sensor, sensor: dict) -> dict:
        """Projection mapping (R14): ALLOCATE as integrate, then every voxel of
        the submap is projected into the depth image (nearest pixel) and fused with sdf = depth - z."""
        d = np.ascontiguousarray(np.asarray(depth, dtype=np.float32))
        T = np.ascontiguousarray(T_world_sensor, dtype=np.float64)
        st = Stats()
        sm = sensor_struct(sensor)
        rc = lib().orc_integrate_projective(self._h, _p(d), d.size, _p(T), C.byref(sm), C.byref(st))
        assert rc == 0, "projective integration needs a pinhole depth frame of width*height pixels"
        return st.asdict()

    def num_blocks(self) -> int:
        return int(lib().orc_num_blocks(self._h))

    def integrate_color(self, data, rgb, T_world_sensor, sensor: dict) -> dict:
        """TSDF + Color (R13): as integrate, plus uint8 rgb [n, 3] per point."""
        d = np.ascontiguousarray(np.asarray(data, dtype=np.float32))
        n = d.size if sensor["kind"] == 1 else d.size // 3
        c = np.ascontiguousarray(np.asarray(rgb, dtype=np.uint8))
        assert c.size == 3 * n
        T = np.ascontiguousarray(T_world_sensor, dtype=np.float64)
        sm = sensor_struct(sensor)
        st = Stats()
        rc = lib().orc_integrate_color(self._h, _p(d), _p(c), n, _p(T), C.byref(sm), C.byref(st))
        assert rc == 0
        return st.asdict()

    def export_color(self):
        """(rgb fp64 [nb,512,3], colour weight fp64 [nb,512]) in the order of export()."""
        nb = self.num_blocks()
        rgb = np.zeros((nb, 512, 3))
        cw = np.zeros((nb, 512))
        lib().orc_export_color(self._h, _p(rgb), _p(cw))
        return rgb, cw

    def export(self):
        """(bxyz int32 [nb,3], D fp64 [nb,512], W fp64 [nb,512]) in lexicographic (bx,by,bz) order."""
        nb = self.num_blocks()
        b = np.zeros((nb, 3), np.int32)
        D = np.zeros((nb, 512), np.float64)
        W = np.zeros((nb, 512), np.float64)
        if nb:
            lib().orc_export(self._h, _p(b), _p(D), _p(W))
        return b, D, W


def project_voxels(grid: dict, T_world_submap, depth, T_world_sensor, sensor: dict, voxels):
    """Projective sums (swd, sw) fp64 [m] of listed voxels [m,3] over all frames (R14 step 2 per voxel;
    for voxels whose block exists from the first frame on)."""
    g = grid_struct(grid)
    Tws = np.ascontiguousarray(T_world_submap, dtype=np.float64)
    d = np.ascontiguousarray(np.asarray(depth, dtype=np.float32))
    T = np.ascontiguousarray(np.asarray(T_world_sensor, dtype=np.float64).reshape(-1, 16))
    v = np.ascontiguousarray(voxels, dtype=np.int32)
    m = v.shape[0]
    swd = np.zeros(m)
    sw = np.zeros(m)
    lib().orc_project_voxels(C.byref(g), _p(Tws), _p(d), T.shape[0], _p(T), C.byref(sensor_struct(sensor)), _p(v), m,
                             _p(swd), _p(sw))
    return swd, sw


def ray_voxels(o, p, voxel_size: float, truncation: float, carve: int = 1) -> np.ndarray:
    """Ordered voxel list [n,3] of one ray (O3-O4); None when outside the key domain."""
    o = np.ascontiguousarray(o, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    cap = 1 << 16
    out = np.zeros((cap, 3), np.int32)
    n = lib().orc_ray_voxels(_p(o), _p(p), voxel_size, truncation, carve, _p(out), cap)
    if n < 0:
        return None
    assert n <= cap
    return out[:n].copy()


def esdf(bxyz, D, W, voxel_size: float, site_threshold: float, brute: bool = False):
    """(E fp64 [nb,512], d2 int64 [nb,512] with -1 = no site) per O10-O12."""
    b = np.ascontiguousarray(bxyz, dtype=np.int32)
    Dd = np.ascontiguousarray(D, dtype=np.float64)
    Wd = np.ascontiguousarray(W, dtype=np.float64)
    nb = b.shape[0]
    E = np.zeros((nb, 512), np.float64)
    d2 = np.zeros((nb, 512), np.int64)
    if nb:
        rc = lib().orc_esdf(_p(b), _p(Dd), _p(Wd), nb, voxel_size, site_threshold, int(brute), _p(E), _p(d2))
        assert rc == 0
    return E, d2


def esdf_capped(bxyz, D, W, voxel_size: float, site_threshold: float, max_distance: float, brute: bool = False):
    """E fp64 [nb,512] of the incremental ESDF (f1, R11): O11 clamped at max_distance."""
    b = np.ascontiguousarray(bxyz, dtype=np.int32)
    Dd = np.ascontiguousarray(D, dtype=np.float64)
    Wd = np.ascontiguousarray(W, dtype=np.float64)
    nb = b.shape[0]
    E = np.zeros((nb, 512), np.float64)
    if nb:
        rc = lib().orc_esdf_capped(_p(b), _p(Dd), _p(Wd), nb, voxel_size, site_threshold, max_distance, int(brute),
                                   _p(E))
        assert rc == 0
    return E


def esdf_sample(bxyz, D, W, site_threshold: float, voxels):
    """Brute-force squared distance (voxel units) of each sample voxel [m,3] to the nearest site; -1 = none."""
    b = np.ascontiguousarray(bxyz, dtype=np.int32)
    Dd = np.ascontiguousarray(D, dtype=np.float64)
    Wd = np.ascontiguousarray(W, dtype=np.float64)
    v = np.ascontiguousarray(voxels, dtype=np.int64)
    out = np.zeros(v.shape[0], np.int64)
    rc = lib().orc_esdf_sample(_p(b), _p(Dd), _p(Wd), b.shape[0], site_threshold, _p(v), v.shape[0], _p(out))
    assert rc == 0
    return out


def query(bxyz, E, voxel_size: float, T_world_submap, pts, gradient: bool = False):
    """(value fp64 [m], status uint8 [m]) per O13; with gradient=True also the world-frame gradient [m,3]."""
    b = np.ascontiguousarray(bxyz, dtype=np.int32)
    Ed = np.ascontiguousarray(E, dtype=np.float64)
    T = np.ascontiguousarray(T_world_submap, dtype=np.float64)
    x = np.ascontiguousarray(pts, dtype=np.float32)
    m = x.shape[0]
    out = np.zeros(m, np.float64)
    st = np.zeros(m, np.uint8)
    g = np.zeros((m, 3), np.float64) if gradient else None
    rc = lib().orc_query(_p(b), _p(Ed), b.shape[0], voxel_size, _p(T), _p(x), m, _p(out), _p(st),
                         _p(g) if gradient else None)
    assert rc == 0
    return (out, st, g) if gradient else (out, st)


def sample_surface(bxyz, D, W, site_threshold: float, voxel_size: float, T_world_submap, uniforms):
    """(xyz fp32 [m,3], weight fp64 [m], total) per DESIGN.md R12 (f4)."""
    b = np.ascontiguousarray(bxyz, dtype=np.int32)
    Dd = np.ascontiguousarray(D, dtype=np.float64)
    Wd = np.ascontiguousarray(W, dtype=np.float64)
    T = np.ascontiguousarray(T_world_submap, dtype=np.float64)
    u = np.ascontiguousarray(uniforms, dtype=np.uint32)
    m = u.shape[0]
    xyz = np.zeros((m, 3), np.float32)
    w = np.zeros(m, np.float64)
    tot = np.zeros(1, np.uint64)
    rc = lib().orc_sample_surface(_p(b), _p(Dd), _p(Wd), b.shape[0], site_threshold, voxel_size, _p(T), _p(u), m,
                                  _p(xyz), _p(w), _p(tot))
    assert rc == 0
    return xyz, w, int(tot[0])


def build_submap(cfg: dict, submap: int = 0, frames=None) -> tuple[OracleSubmap, list]:
    """Integrate (a subset of) one config submap's frames through the oracle."""
    sm = cfg["submaps"][submap]
    o = OracleSubmap(cfg["grid"], sm["T_world_submap"])
    stats = []
    for k in (sm["frames"] if frames is None else frames):
        fr = cfg["frames"][k]
        stats.append(o.integrate(fr["data"].cpu().numpy(), fr["T_world_sensor"], cfg["sensor"]))
    return o, stats
