"""Shared test helpers: run a config through the GPU path (C-ABI) and through the oracle, compare."""
from __future__ import annotations

import numpy as np
import torch

TOL_D = 1e-4      # m   (BASELINE.json north_star: TSDF distances)
TOL_W = 1e-3      # relative, |dW| <= 1e-3 * max(1, W)  (Q22)
TOL_E = 1e-4      # m   (ESDF distances)


def sort_blocks(b, *arrs):
    b = np.asarray(b)
    order = np.lexsort((b[:, 2], b[:, 1], b[:, 0]))
    return (b[order],) + tuple(None if a is None else np.asarray(a)[order] for a in arrs)


def gpu_build(cfg, frames, device=0, batch=False, grid=None, T_ws=None, finalize=True, stats=True):
    from paper_2410_21149_b200 import Submap
    g = dict(cfg["grid"] if grid is None else grid)
    T = cfg["submaps"][0]["T_world_submap"] if T_ws is None else T_ws
    sm = Submap(g, T, device)
    dev = torch.device("cuda", device)
    st = None
    if batch:
        data = torch.stack([cfg["frames"][k]["data"] for k in frames]).to(dev)
        poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in frames])
        st = sm.integrate_batch(data, poses, cfg["sensor"], stats=stats)
    else:
        for k in frames:
            st = sm.integrate(cfg["frames"][k]["data"].to(dev).contiguous(), cfg["frames"][k]["T_world_sensor"],
                              cfg["sensor"], stats=stats)
    if finalize:
        sm.finalize_esdf()
    return sm, st


def gpu_export_sorted(sm):
    b, D, W, E = sm.export(with_esdf=True)
    torch.cuda.synchronize()
    return sort_blocks(b.cpu().numpy(), D.cpu().numpy(), W.cpu().numpy(), E.cpu().numpy())


def oracle_build(cfg, frames, grid=None, T_ws=None):
    import oracle
    g = dict(cfg["grid"] if grid is None else grid)
    T = cfg["submaps"][0]["T_world_submap"] if T_ws is None else T_ws
    o = oracle.OracleSubmap(g, T)
    st = None
    for k in frames:
        st = o.integrate(cfg["frames"][k]["data"].cpu().numpy(), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
    return o, st


def assert_tsdf_parity(gpu_sorted, orc_export):
    bg, Dg, Wg, _ = gpu_sorted
    bo, Do, Wo = orc_export
    assert bg.shape == bo.shape, f"block count gpu {bg.shape[0]} vs oracle {bo.shape[0]}"
    assert np.array_equal(bg, bo), "block sets differ"
    obs_g, obs_o = Wg > 0, Wo > 0
    assert np.array_equal(obs_g, obs_o), f"observed sets differ in {(obs_g != obs_o).sum()} voxels"
    dD = np.abs(Dg.astype(np.float64) - Do)[obs_o]
    dW = np.abs(Wg.astype(np.float64) - Wo)[obs_o] / np.maximum(1.0, Wo[obs_o])
    assert dD.max(initial=0) <= TOL_D, f"max |dD| = {dD.max()}"
    assert dW.max(initial=0) <= TOL_W, f"max rel |dW| = {dW.max()}"
    return dict(blocks=int(bg.shape[0]), observed=int(obs_o.sum()), max_dD=float(dD.max(initial=0)),
                max_dW=float(dW.max(initial=0)))


def assert_esdf_parity(Eg, Eo, obs):
    Eg = Eg.astype(np.float64)
    assert np.array_equal(np.isnan(Eg), np.isnan(Eo)), "NaN pattern differs"
    assert np.array_equal(np.isposinf(Eg), np.isposinf(Eo)), "+inf pattern differs"
    fin = np.isfinite(Eo)
    d = np.abs(Eg[fin] - Eo[fin])
    assert d.max(initial=0) <= TOL_E, f"max |dE| = {d.max()}"
    return float(d.max(initial=0))
