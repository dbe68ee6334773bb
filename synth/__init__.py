"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NONE of the method's arithmetic (no traversal, no SDF, no fusion, no
EDT). It only produces posed sensor data by intersecting analytic rays with analytic
scenes, with the shapes of the paper's workloads (§IV: Ouster OS1
LiDAR MAV flights and Replica/Redwood RGB-D rooms).  Recipes: DESIGN.md "Input recipe".
"""
from .scenes import (  # noqa: F401
    Scene, raycast, make_config, CONFIGS, lidar_directions, pinhole_depth, lidar_scan, camera_pose,
    pose, rot_zyx, surface_color,
)
