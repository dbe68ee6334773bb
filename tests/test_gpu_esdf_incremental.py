"""Incremental ESDF (R11) against the oracle of its value.

The value cvx_update_esdf keeps is the exact EDT of O11 clamped at d_max = grid['esdf_max_distance']
(oracle: orc_esdf_capped, pinned in tests/test_oracle_esdf_query.py).  Stage-isolated like the finalize
parity: the oracle runs on the GPU's exported TSDF, so both see the same sites.  Bar: identical NaN
pattern and |dE| <= 1e-4 m on EVERY voxel, after every update of every schedule; and the result does not
depend on the schedule (bit-identical ESDFs whether updated after every frame or once).
"""
import numpy as np
import pytest
import torch

import synth
from helpers import TOL_E, gpu_export_sorted

pytestmark = pytest.mark.gpu


def _check(sm, orc, grid):
    b, D, W, E = gpu_export_sorted(sm)
    Eo = orc.esdf_capped(b, D.astype(np.float64), W.astype(np.float64), grid["voxel_size"], grid["site_threshold"],
                         grid["esdf_max_distance"])
    Ei = E.astype(np.float64)
    assert np.array_equal(np.isnan(Ei), np.isnan(Eo)), "NaN pattern differs"
    obs = ~np.isnan(Eo)
    d = np.abs(Ei[obs] - Eo[obs])
    assert d.max(initial=0) <= TOL_E, f"max |dE| = {d.max()}"
    assert np.array_equal(np.signbit(Ei[obs]), np.signbit(Eo[obs]))
    return b, E


def _integrate(sm, cfg, k, dev):
    sm.integrate(cfg["frames"][k]["data"].to(dev), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])


@pytest.mark.parametrize("name,frames,every,dmax", [
    ("tiny", list(range(10)), 1, 0.5),      # r = 5 voxels (1 block radius)
    ("tiny", list(range(10)), 4, 1.2),      # r = 12 (2 blocks)
    ("lidar", list(range(0, 40, 2)), 10, 2.0),  # configs[1] geometry, 20 scans, an update every 10
])
def test_incremental_matches_capped_oracle(orc, name, frames, every, dmax):
    cfg = synth.make_config(name, frames=frames)
    grid = dict(cfg["grid"], esdf_max_distance=dmax)
    from paper_2410_21149_b200 import Submap
    dev = torch.device("cuda", 0)
    sm = Submap(grid, cfg["submaps"][0]["T_world_submap"], 0)
    nq = []
    for i, k in enumerate(frames):
        _integrate(sm, cfg, k, dev)
        if (i + 1) % every == 0 or i + 1 == len(frames):
            nq.append(sm.update_esdf())
            _check(sm, orc, grid)
    assert nq[0] == sm.block_count() or len(nq) == 1 or nq[0] > 0
    # one update at the end gives the same ESDF bit for bit (schedule independence)
    once = Submap(grid, cfg["submaps"][0]["T_world_submap"], 0)
    for k in frames:
        _integrate(once, cfg, k, dev)
    assert once.update_esdf() == once.block_count()
    e1, e2 = gpu_export_sorted(sm)[3], gpu_export_sorted(once)[3]
    assert np.array_equal(e1.view(np.uint32), e2.view(np.uint32))
    d, s = sm.query(torch.zeros((8, 3), device=dev))          # queries work on the incremental ESDF
    assert s.shape[0] == 8


def test_incremental_nothing_changed_and_raise(orc):
    """No change -> no block recomputed and the ESDF is untouched; removing sites (raise) and
    adding sites (lower) through TSDF imports -> every voxel matches the clamped oracle again."""
    from paper_2410_21149_b200 import Submap
    rng = np.random.default_rng(7)
    dev = torch.device("cuda", 0)
    blocks = np.array([(x, y, z) for x in range(-3, 3) for y in range(-2, 3) for z in range(-1, 2)], np.int32)
    nb = len(blocks)
    W = ((rng.random((nb, 512)) < 0.9) * rng.uniform(0.5, 2, (nb, 512))).astype(np.float32)
    D = (rng.uniform(-0.3, 0.3, (nb, 512)) * (W > 0)).astype(np.float32)
    D[np.abs(D) <= 0.01] = 0.2                                  # start without sites ...
    D[3, 100] = 0.0; D[40, 7] = -0.005; D[70, 300] = 0.003       # ... except three
    grid = dict(voxel_size=0.1, truncation=0.3, site_threshold=0.01, max_blocks=4096, esdf_max_distance=0.75)
    sm = Submap(grid)
    t = lambda a: torch.from_numpy(a).to(dev)
    sm.import_tsdf(t(blocks), t(D), t(W))
    assert sm.update_esdf() == nb
    _check(sm, orc, grid)
    e0 = gpu_export_sorted(sm)[3]
    assert sm.update_esdf() == 0
    assert np.array_equal(e0.view(np.uint32), gpu_export_sorted(sm)[3].view(np.uint32))
    # raise: remove the site of block 40; lower: add a site far from the others; flip an observation
    D2, W2 = D.copy(), W.copy()
    D2[40, 7] = 0.25
    D2[10, 511] = 0.0; W2[10, 511] = 1.0
    W2[60, :64] = 0.0; D2[60, :64] = 0.0
    sel = np.array([40, 10, 60])
    sm.import_tsdf(t(blocks[sel]), t(D2[sel]), t(W2[sel]))
    n = sm.update_esdf()
    assert 0 < n < nb
    _check(sm, orc, grid)
    # the result equals a fresh submap updated once
    fresh = Submap(grid)
    fresh.import_tsdf(t(blocks), t(D2), t(W2))
    fresh.update_esdf()
    assert np.array_equal(gpu_export_sorted(sm)[3].view(np.uint32), gpu_export_sorted(fresh)[3].view(np.uint32))


def test_incremental_wide_window_uses_dense_path(orc):
    """d_max > 24 voxels: the window would exceed 7^3 blocks, so the update runs the dense exact EDT with
    the clamp — same value definition, checked against the oracle on every voxel."""
    cfg = synth.make_config("tiny", frames=[0, 3, 6])
    grid = dict(cfg["grid"], esdf_max_distance=3.0)           # 30 voxels at 0.1 m
    from paper_2410_21149_b200 import Submap
    dev = torch.device("cuda", 0)
    sm = Submap(grid, cfg["submaps"][0]["T_world_submap"], 0)
    for k in (0, 3):
        _integrate(sm, cfg, k, dev)
    assert sm.update_esdf() == sm.block_count()
    _check(sm, orc, grid)
    _integrate(sm, cfg, 6, dev)
    sm.update_esdf()
    _check(sm, orc, grid)


def test_finalize_after_incremental_is_exact(orc):
    """finalize_esdf after incremental updates gives the exact unclamped O11 (and a later update
    recomputes every block of the clamped ESDF)."""
    cfg = synth.make_config("tiny", frames=[0, 2, 4])
    grid = dict(cfg["grid"], esdf_max_distance=0.4)
    from paper_2410_21149_b200 import Submap
    dev = torch.device("cuda", 0)
    sm = Submap(grid, cfg["submaps"][0]["T_world_submap"], 0)
    for k in (0, 2, 4):
        _integrate(sm, cfg, k, dev)
        sm.update_esdf()
    sm.finalize_esdf()
    b, D, W, E = gpu_export_sorted(sm)
    Eo, _ = orc.esdf(b, D.astype(np.float64), W.astype(np.float64), grid["voxel_size"], grid["site_threshold"])
    fin = np.isfinite(Eo)
    assert np.array_equal(np.isnan(E), np.isnan(Eo))
    assert np.abs(E[fin] - Eo[fin]).max() <= TOL_E
    assert sm.update_esdf() == sm.block_count()
    _check(sm, orc, grid)
