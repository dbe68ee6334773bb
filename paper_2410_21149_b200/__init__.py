"""B200-native coVoxSLAM submap builder (arXiv 2410.21149): block-hashed TSDF fusion by raycasting,
exact ESDF, distance queries — hand-written sm_100a CUDA behind the C-ABI in include/cvx.h.

The Python surface is a thin ctypes binding (cvx.py); it never computes any step of the method.
"""
from .cvx import (  # noqa: F401
    Submap, EsdfSet, CvxError, lib, unpack, payload_bytes, STATUS_OK, STATUS_NEAREST, STATUS_UNKNOWN, SIGNATURES,
)
