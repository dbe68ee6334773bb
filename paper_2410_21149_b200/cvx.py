"""Thin Python binding of libcvx (include/cvx.h): argument marshalling only.

Every step of the submap build runs in libcvx's sm_100a kernels; this module only checks tensor
placement/dtype, passes raw device pointers, the current torch stream and host poses through the
C-ABI, and turns error codes into exceptions.  There is no CPU fallback: if libcvx.so is missing or
cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# CVX_LIB_PATH: load another build of the same library (the bounds-checked build of tests/test_gpu_bounds.py)
LIB_PATH = os.environ.get("CVX_LIB_PATH") or os.path.join(_HERE, "libcvx.so")

OK, E_INVALID, E_OOM, E_CAPACITY, E_STATE, E_CUDA, E_RANGE = 0, -1, -2, -3, -4, -5, -6
_NAMES = {E_INVALID: "CVX_E_INVALID", E_OOM: "CVX_E_OOM", E_CAPACITY: "CVX_E_CAPACITY",
          E_STATE: "CVX_E_STATE", E_CUDA: "CVX_E_CUDA", E_RANGE: "CVX_E_RANGE"}
STATUS_OK, STATUS_NEAREST, STATUS_UNKNOWN = 0, 1, 2
RECORD_BYTES = 16 + 4 * 512
HEADER_BYTES = 256


class CvxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class GridConfig(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("block_side", C.c_int32), ("truncation", C.c_double),
                ("weighting", C.c_int32), ("weight_range_floor", C.c_double), ("carve", C.c_int32),
                ("site_threshold", C.c_double), ("max_blocks", C.c_int64), ("color", C.c_int32),
                ("esdf_max_distance", C.c_double)]


class SensorModel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("min_range", C.c_float), ("max_range", C.c_float)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("rays_in", "rays_used", "skipped_invalid", "skipped_range",
                                         "skipped_domain", "voxel_updates", "new_blocks", "total_blocks")]

    def asdict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


# every symbol include/cvx.h declares, with its ctypes signature
_P = C.c_void_p
SIGNATURES = {
    "cvx_create_submap": (C.c_int32, [C.POINTER(GridConfig), _P, C.c_int, C.POINTER(_P)]),
    "cvx_destroy_submap": (C.c_int32, [_P]),
    "cvx_reset_submap": (C.c_int32, [_P, _P]),
    "cvx_set_submap_pose": (C.c_int32, [_P, _P]),
    "cvx_integrate_pointcloud": (C.c_int32, [_P, _P, C.c_int64, _P, C.POINTER(SensorModel), _P, C.POINTER(Stats)]),
    "cvx_integrate_batch": (C.c_int32, [_P, _P, C.c_int64, C.c_int32, _P, C.POINTER(SensorModel), _P,
                                        C.POINTER(Stats)]),
    "cvx_integrate_batch_host": (C.c_int32, [_P, _P, C.c_int64, C.c_int32, _P, C.POINTER(SensorModel), _P,
                                             C.POINTER(Stats)]),
    "cvx_integrate_until": (C.c_int32, [_P, _P, C.c_int64, C.c_int32, _P, C.POINTER(SensorModel), C.c_int64, _P,
                                        C.POINTER(C.c_int32)]),
    "cvx_integrate_color": (C.c_int32, [_P, _P, _P, C.c_int64, C.c_int32, _P, C.POINTER(SensorModel), _P,
                                        C.POINTER(Stats)]),
    "cvx_integrate_projective": (C.c_int32, [_P, _P, C.c_int64, C.c_int32, _P, C.POINTER(SensorModel), _P,
                                             C.POINTER(Stats)]),
    "cvx_export_color": (C.c_int32, [_P, _P, _P, C.c_int64, C.POINTER(C.c_int64), _P]),
    "cvx_get_stats": (C.c_int32, [_P, C.POINTER(Stats)]),
    "cvx_get_block_count": (C.c_int32, [_P, C.POINTER(C.c_int64)]),
    "cvx_get_aabb": (C.c_int32, [_P, _P, _P]),
    "cvx_finalize_esdf": (C.c_int32, [_P, _P]),
    "cvx_update_esdf": (C.c_int32, [_P, _P, C.POINTER(C.c_int32)]),
    "cvx_query_distance": (C.c_int32, [_P, _P, C.c_int64, _P, _P, _P]),
    "cvx_query_distance_gradient": (C.c_int32, [_P, _P, C.c_int64, _P, _P, _P, _P]),
    "cvx_sample_surface": (C.c_int32, [_P, _P, C.c_int64, _P, _P, C.POINTER(C.c_int64), _P]),
    "cvx_export_blocks": (C.c_int32, [_P, _P, _P, _P, _P, C.c_int64, C.POINTER(C.c_int64), _P]),
    "cvx_import_tsdf_blocks": (C.c_int32, [_P, _P, _P, _P, C.c_int64, _P]),
    "cvx_pack_esdf": (C.c_int32, [_P, _P, C.c_int64, C.POINTER(C.c_int64), _P]),
    "cvx_packed_size": (C.c_int32, [_P, C.POINTER(C.c_int64)]),
    "cvx_esdf_set_create": (C.c_int32, [_P, C.c_int64, _P, C.c_int32, C.c_int, _P, C.POINTER(_P)]),
    "cvx_esdf_set_destroy": (C.c_int32, [_P]),
    "cvx_esdf_set_query": (C.c_int32, [_P, _P, _P, C.c_int64, _P, _P, _P, _P]),
    "cvx_profile_enable": (C.c_int32, [_P, C.c_int32]),
    "cvx_profile_report": (C.c_int32, [_P, C.c_char_p, C.c_int64]),
    "cvx_last_error": (C.c_char_p, []),
    "cvx_version": (C.c_char_p, []),
}

_lib = None


def lib():
    """Load libcvx.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libcvx.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise CvxError(rc, lib().cvx_last_error().decode())


def _pose(T) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(T, dtype=np.float64).reshape(-1, 16))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def grid_config(grid: dict) -> GridConfig:
    return GridConfig(float(grid["voxel_size"]), int(grid.get("block_side", 8)), float(grid["truncation"]),
                      int(grid.get("weighting", 0)), float(grid.get("weight_range_floor", 0.1)),
                      int(grid.get("carve", 1)), float(grid.get("site_threshold", grid["voxel_size"])),
                      int(grid.get("max_blocks", 1 << 16)), int(grid.get("color", 0)),
                      float(grid.get("esdf_max_distance", 2.0)))


def sensor_model(sensor: dict) -> SensorModel:
    return SensorModel(int(sensor["kind"]), int(sensor.get("width", 0)), int(sensor.get("height", 0)),
                       float(sensor.get("fx", 0)), float(sensor.get("fy", 0)), float(sensor.get("cx", 0)),
                       float(sensor.get("cy", 0)), float(sensor.get("min_range", 0.0)),
                       float(sensor.get("max_range", 3.0e38)))


class Submap:
    """One submap on one CUDA device (cvx_submap)."""

    def __init__(self, grid: dict, T_world_submap=None, device: int = 0):
        self.grid = dict(grid)
        self.device = int(device)
        self.T_ws = _pose(np.eye(4) if T_world_submap is None else T_world_submap)[0].reshape(4, 4).copy()
        self._cfg = grid_config(grid)
        h = C.c_void_p()
        _check(lib().cvx_create_submap(C.byref(self._cfg), _ptr(_pose(self.T_ws)), self.device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().cvx_destroy_submap(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers -------------------------------------------------------------------------------
    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _dev(self, t: torch.Tensor, dtype, name):
        if not (t.is_cuda and t.device.index == self.device):
            raise ValueError(f"{name} must be a CUDA tensor on cuda:{self.device}")
        if t.dtype != dtype:
            raise TypeError(f"{name} must be {dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        return C.c_void_p(t.data_ptr())

    # -- the four calls --------------------------------------------------------------------------
    def integrate(self, data: torch.Tensor, T_world_sensor, sensor: dict, stats: bool = False):
        sm = sensor_model(sensor)
        n = data.numel() if sensor["kind"] == 1 else data.numel() // 3
        st = Stats() if stats else None
        _check(lib().cvx_integrate_pointcloud(self._h, self._dev(data, torch.float32, "data"), n,
                                              _ptr(_pose(T_world_sensor)), C.byref(sm), self._stream(),
                                              C.byref(st) if st is not None else None))
        return st.asdict() if st is not None else None

    def integrate_batch(self, data: torch.Tensor, T_world_sensor, sensor: dict, stats: bool = False):
        """data: [F, n, 3] points or [F, H, W] depth; T_world_sensor: [F, 4, 4]."""
        sm = sensor_model(sensor)
        F = data.shape[0]
        n = data[0].numel() if sensor["kind"] == 1 else data[0].numel() // 3
        poses = _pose(T_world_sensor)
        if poses.shape[0] != F:
            raise ValueError("one pose per frame")
        st = Stats() if stats else None
        _check(lib().cvx_integrate_batch(self._h, self._dev(data, torch.float32, "data"), n, F, _ptr(poses),
                                         C.byref(sm), self._stream(), C.byref(st) if st is not None else None))
        return st.asdict() if st is not None else None

    def integrate_projective(self, depth: torch.Tensor, T_world_sensor, sensor: dict, stats: bool = False):
        """Projection mapping (R14): depth fp32 [F, H, W] (or [H, W]),
        T_world_sensor [F, 4, 4]; pinhole sensors only."""
        if depth.dim() == 2:
            depth = depth.unsqueeze(0)
        sm = sensor_model(sensor)
        F = depth.shape[0]
        poses = _pose(T_world_sensor)
        if poses.shape[0] != F:
            raise ValueError("one pose per frame")
        st = Stats() if stats else None
        _check(lib().cvx_integrate_projective(self._h, self._dev(depth, torch.float32, "depth"), depth[0].numel(), F,
                                              _ptr(poses), C.byref(sm), self._stream(),
                                              C.byref(st) if st is not None else None))
        return st.asdict() if st is not None else None

    def integrate_color(self, data: torch.Tensor, rgb: torch.Tensor, T_world_sensor, sensor: dict,
                        stats: bool = False):
        """TSDF + Color: data as integrate_batch, rgb uint8 [F, n, 3] (same point order)."""
        sm = sensor_model(sensor)
        F = data.shape[0]
        n = data[0].numel() if sensor["kind"] == 1 else data[0].numel() // 3
        if rgb.numel() != F * n * 3:
            raise ValueError("rgb must hold 3 bytes per point")
        poses = _pose(T_world_sensor)
        if poses.shape[0] != F:
            raise ValueError("one pose per frame")
        st = Stats() if stats else None
        _check(lib().cvx_integrate_color(self._h, self._dev(data, torch.float32, "data"),
                                         self._dev(rgb, torch.uint8, "rgb"), n, F, _ptr(poses), C.byref(sm),
                                         self._stream(), C.byref(st) if st is not None else None))
        return st.asdict() if st is not None else None

    def export_color(self):
        """(rgb fp32 [nb,512,3] in 0..255, colour weight fp32 [nb,512]), slot order (as export())."""
        nb = self.block_count()
        dev = torch.device("cuda", self.device)
        rgb = torch.empty((nb, 512, 3), dtype=torch.float32, device=dev)
        cw = torch.empty((nb, 512), dtype=torch.float32, device=dev)
        n = C.c_int64()
        _check(lib().cvx_export_color(self._h, C.c_void_p(rgb.data_ptr()), C.c_void_p(cw.data_ptr()), nb,
                                      C.byref(n), self._stream()))
        return rgb, cw

    def integrate_until(self, data: torch.Tensor, T_world_sensor, sensor: dict, block_threshold: int) -> int:
        """Integrate frames until the submap holds >= block_threshold blocks; returns the frames taken."""
        sm = sensor_model(sensor)
        F = data.shape[0]
        n = data[0].numel() if sensor["kind"] == 1 else data[0].numel() // 3
        poses = _pose(T_world_sensor)
        if poses.shape[0] != F:
            raise ValueError("one pose per frame")
        k = C.c_int32()
        _check(lib().cvx_integrate_until(self._h, self._dev(data, torch.float32, "data"), n, F, _ptr(poses), C.byref(sm),
                                         int(block_threshold), self._stream(), C.byref(k)))
        return int(k.value)

    def integrate_batch_host(self, data: torch.Tensor, T_world_sensor, sensor: dict, stats: bool = False):
        """Like integrate_batch with `data` a CPU tensor (pin_memory() for asynchronous copies)."""
        if data.is_cuda or data.dtype != torch.float32 or not data.is_contiguous():
            raise ValueError("data must be a contiguous float32 CPU tensor")
        sm = sensor_model(sensor)
        F = data.shape[0]
        n = data[0].numel() if sensor["kind"] == 1 else data[0].numel() // 3
        poses = _pose(T_world_sensor)
        if poses.shape[0] != F:
            raise ValueError("one pose per frame")
        st = Stats() if stats else None
        _check(lib().cvx_integrate_batch_host(self._h, C.c_void_p(data.data_ptr()), n, F, _ptr(poses), C.byref(sm),
                                              self._stream(), C.byref(st) if st is not None else None))
        return st.asdict() if st is not None else None

    def finalize_esdf(self):
        _check(lib().cvx_finalize_esdf(self._h, self._stream()))

    def update_esdf(self) -> int:
        """Incremental ESDF update (cvx_update_esdf): the exact ESDF clamped at grid['esdf_max_distance'];
        returns the number of blocks recomputed."""
        it = C.c_int32()
        _check(lib().cvx_update_esdf(self._h, self._stream(), C.byref(it)))
        return int(it.value)

    def query(self, points_world: torch.Tensor, out: torch.Tensor | None = None,
              status: torch.Tensor | None = None):
        m = points_world.shape[0]
        if out is None:
            out = torch.empty(m, dtype=torch.float32, device=points_world.device)
        if status is None:
            status = torch.empty(m, dtype=torch.uint8, device=points_world.device)
        _check(lib().cvx_query_distance(self._h, self._dev(points_world, torch.float32, "points"), m,
                                        self._dev(out, torch.float32, "out"),
                                        self._dev(status, torch.uint8, "status"), self._stream()))
        return out, status

    def query_gradient(self, points_world: torch.Tensor):
        """(distance [m], gradient [m,3] world frame, status [m]) — cvx_query_distance_gradient."""
        m = points_world.shape[0]
        dev = points_world.device
        out = torch.empty(m, dtype=torch.float32, device=dev)
        grad = torch.empty((m, 3), dtype=torch.float32, device=dev)
        status = torch.empty(m, dtype=torch.uint8, device=dev)
        _check(lib().cvx_query_distance_gradient(self._h, self._dev(points_world, torch.float32, "points"), m,
                                                 self._dev(out, torch.float32, "out"),
                                                 self._dev(grad, torch.float32, "grad"),
                                                 self._dev(status, torch.uint8, "status"), self._stream()))
        return out, grad, status

    def sample_surface(self, uniforms: torch.Tensor):
        """(xyz [m,3] world, weight [m], total weight) for uint32 uniforms [m] (int32 tensor bit patterns)."""
        m = uniforms.shape[0]
        dev = uniforms.device
        xyz = torch.empty((m, 3), dtype=torch.float32, device=dev)
        w = torch.empty(m, dtype=torch.float32, device=dev)
        tot = C.c_int64()
        _check(lib().cvx_sample_surface(self._h, self._dev(uniforms, torch.int32, "uniforms"), m,
                                        self._dev(xyz, torch.float32, "xyz"), self._dev(w, torch.float32, "w"),
                                        C.byref(tot), self._stream()))
        return xyz, w, int(tot.value)

    # -- state / inspection --------------------------------------------------------------------
    def reset(self, T_world_submap=None):
        """Empty the submap (cvx_reset_submap); optionally give it a new pose (cvx_set_submap_pose)."""
        _check(lib().cvx_reset_submap(self._h, self._stream()))
        if T_world_submap is not None:
            T = _pose(T_world_submap)
            _check(lib().cvx_set_submap_pose(self._h, _ptr(T)))
            self.T_ws = T[0].reshape(4, 4).copy()

    def stats(self) -> dict:
        torch.cuda.current_stream(self.device).synchronize()
        st = Stats()
        _check(lib().cvx_get_stats(self._h, C.byref(st)))
        return st.asdict()

    def block_count(self) -> int:
        torch.cuda.current_stream(self.device).synchronize()
        n = C.c_int64()
        _check(lib().cvx_get_block_count(self._h, C.byref(n)))
        return int(n.value)

    def aabb(self):
        torch.cuda.current_stream(self.device).synchronize()
        lo = np.zeros(3, np.int32)
        hi = np.zeros(3, np.int32)
        _check(lib().cvx_get_aabb(self._h, _ptr(lo), _ptr(hi)))
        return lo, hi

    def export(self, with_esdf: bool = True):
        """(bxyz int32 [nb,3], D fp32 [nb,512], W fp32 [nb,512], E fp32 [nb,512] | None), slot order."""
        nb = self.block_count()
        dev = torch.device("cuda", self.device)
        b = torch.empty((nb, 3), dtype=torch.int32, device=dev)
        D = torch.empty((nb, 512), dtype=torch.float32, device=dev)
        W = torch.empty((nb, 512), dtype=torch.float32, device=dev)
        E = torch.empty((nb, 512), dtype=torch.float32, device=dev) if with_esdf else None
        n = C.c_int64()
        _check(lib().cvx_export_blocks(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(D.data_ptr()),
                                       C.c_void_p(W.data_ptr()), C.c_void_p(E.data_ptr()) if E is not None else None,
                                       nb, C.byref(n), self._stream()))
        return b, D, W, E

    def import_tsdf(self, bxyz: torch.Tensor, D: torch.Tensor, W: torch.Tensor):
        n = bxyz.shape[0]
        _check(lib().cvx_import_tsdf_blocks(self._h, self._dev(bxyz, torch.int32, "bxyz"),
                                            self._dev(D, torch.float32, "D"), self._dev(W, torch.float32, "W"),
                                            n, self._stream()))

    def profile(self, enable: bool = True, serialize: bool = False):
        """Per-kernel CUDA-event timing; serialize=True also runs the pipeline's side work on the caller's
        stream (solo kernel times)."""
        _check(lib().cvx_profile_enable(self._h, (1 if enable else 0) | (2 if serialize else 0)))

    def profile_report(self) -> dict:
        import json
        buf = C.create_string_buffer(1 << 16)
        _check(lib().cvx_profile_report(self._h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def packed_size(self) -> int:
        torch.cuda.current_stream(self.device).synchronize()
        n = C.c_int64()
        _check(lib().cvx_packed_size(self._h, C.byref(n)))
        return int(n.value)

    def pack(self, dst: torch.Tensor | None = None) -> torch.Tensor:
        used0 = C.c_int64()   # size query ordered on the current stream only (no device-wide sync)
        _check(lib().cvx_pack_esdf(self._h, None, 0, C.byref(used0), self._stream()))
        need = int(used0.value)
        if dst is None:
            dst = torch.empty(need, dtype=torch.uint8, device=torch.device("cuda", self.device))
        used = C.c_int64()
        _check(lib().cvx_pack_esdf(self._h, self._dev(dst, torch.uint8, "dst"), dst.numel(), C.byref(used),
                                   self._stream()))
        return dst[:used.value]


def unpack(buf: torch.Tensor):
    """Parse one cvx_pack_esdf payload -> dict(T_world_submap, voxel_size, bxyz, E). Host-side view only."""
    raw = buf.detach().cpu().numpy().tobytes()
    magic, version, nb = np.frombuffer(raw[:16], dtype=np.dtype([("m", "<u4"), ("v", "<i4"), ("n", "<i8")]))[0]
    if magic != 0x45585643:
        raise ValueError("not a CVXE payload")
    vs = np.frombuffer(raw[16:24], "<f8")[0]
    T = np.frombuffer(raw[24:152], "<f8").reshape(4, 4)
    rec = np.frombuffer(raw[HEADER_BYTES:HEADER_BYTES + nb * RECORD_BYTES], dtype=np.uint8).reshape(nb, RECORD_BYTES)
    hdr = rec[:, :16].copy().view("<i4").reshape(nb, 4)
    E = rec[:, 16:].copy().view("<f4").reshape(nb, 512)
    return dict(T_world_submap=T.copy(), voxel_size=float(vs), bxyz=hdr[:, :3].copy(), E=E)


class EsdfSet:
    """Gathered submap ESDFs (cvx_esdf_set): `payloads` is a CUDA uint8 buffer holding cvx_pack_esdf
    payloads at byte `offsets` (e.g. the all-gathered ESDFs of every rank); queries name a submap per point.
    The set indexes the buffer in place, so it keeps a reference to the tensor."""

    def __init__(self, payloads: torch.Tensor, offsets, device: int | None = None):
        if not (payloads.is_cuda and payloads.dtype == torch.uint8 and payloads.is_contiguous()):
            raise ValueError("payloads must be a contiguous CUDA uint8 tensor")
        self.device = payloads.device.index if device is None else int(device)
        self._buf = payloads
        off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        self.n = int(off.shape[0])
        h = C.c_void_p()
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().cvx_esdf_set_create(C.c_void_p(payloads.data_ptr()), payloads.numel(), _ptr(off), self.n,
                                         self.device, st, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().cvx_esdf_set_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, submap_index: torch.Tensor, points_world: torch.Tensor, gradient: bool = False):
        """(distance [m], status [m]) or, with gradient=True, (distance, gradient [m,3], status)."""
        m = points_world.shape[0]
        dev = points_world.device
        for t, dt, name in ((submap_index, torch.int32, "submap_index"), (points_world, torch.float32, "points")):
            if not (t.is_cuda and t.dtype == dt and t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous CUDA {dt} tensor")
        if submap_index.numel() != m:
            raise ValueError("one submap index per point")
        out = torch.empty(m, dtype=torch.float32, device=dev)
        status = torch.empty(m, dtype=torch.uint8, device=dev)
        grad = torch.empty((m, 3), dtype=torch.float32, device=dev) if gradient else None
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().cvx_esdf_set_query(self._h, C.c_void_p(submap_index.data_ptr()), C.c_void_p(points_world.data_ptr()),
                                        m, C.c_void_p(out.data_ptr()),
                                        C.c_void_p(grad.data_ptr()) if grad is not None else None,
                                        C.c_void_p(status.data_ptr()), st))
        return (out, grad, status) if gradient else (out, status)


def payload_bytes(n_blocks: int) -> int:
    """Size of one cvx_pack_esdf payload of n_blocks blocks (header + records)."""
    return HEADER_BYTES + int(n_blocks) * RECORD_BYTES
