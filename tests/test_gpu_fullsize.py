"""Full-size parity: BASELINE.json configs[1] (200 OS1-64 scans, 0.2 m voxels) in the launch
configuration bench.py times (one integrate_batch of 200 scans = one walk launch of 2^24 - 1 rays at most),
checked element by element against the oracle's full 200-scan build (TSDF and the stage-isolated exact
ESDF), on sampled outputs the oracle computes one by one, and on properties that hold at any size.
"""
import numpy as np
import pytest
import torch

import synth
from helpers import TOL_E, assert_tsdf_parity, gpu_export_sorted, oracle_build, sort_blocks

pytestmark = pytest.mark.gpu

BATCH = 200  # bench.py default (one integrate_batch call; the library runs one walk launch of 200 scans)


@pytest.fixture(scope="module")
def lidar():
    dev = torch.device("cuda", 0)
    cfg = synth.make_config("lidar", device=dev)
    data = torch.stack([cfg["frames"][k]["data"] for k in range(200)]).contiguous()
    poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in range(200)])
    return cfg, data, poses


def _build(cfg, data, poses, batch, finalize=True):
    from paper_2410_21149_b200 import Submap
    sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    for c in range(0, data.shape[0], batch):
        sm.integrate_batch(data[c:c + batch], poses[c:c + batch], cfg["sensor"])
    if finalize:
        sm.finalize_esdf()
    return sm


@pytest.fixture(scope="module")
def built(lidar):
    cfg, data, poses = lidar
    sm = _build(cfg, data, poses, BATCH)
    return sm, gpu_export_sorted(sm), sm.stats()


def test_fullsize_count_identity_and_batch_independence(lidar, built):
    cfg, data, poses = lidar
    sm, (b, D, W, E), st = built
    assert st["rays_in"] == 200 * 65536 and st["total_blocks"] == b.shape[0] > 20000
    # COUNT (closed form, a2) == what UPDATE deposited (constant weights: W counts updates exactly)
    assert W.astype(np.float64).sum() == st["voxel_updates"]
    # exact integer fusion (R1): a different launch grouping gives bit-identical state
    sm7 = _build(cfg, data, poses, 7, finalize=False)
    b7, D7, W7, _ = gpu_export_sorted(sm7)
    assert np.array_equal(b7, b)
    assert np.array_equal(D7.view(np.uint32), D.view(np.uint32)) and np.array_equal(W7.view(np.uint32), W.view(np.uint32))


@pytest.mark.parametrize("knob", ["CVX_DENSE=0", "CVX_DENSE_BLOCKS=100000"])
def test_fullsize_dense_window_equals_slot_list_path(lidar, built, monkeypatch, knob):
    """DESIGN.md R19 at full size: the default dense-window path (ALLOCATE after the walk) and the slot-list
    path — chosen on the host (CVX_DENSE=0) or by the device-side fallback, with a window buffer (1e5
    blocks) smaller than the launch's box (~2.3e5 blocks) — give the same blocks and the same TSDF bit for
    bit."""
    cfg, data, poses = lidar
    _, (b, D, W, _), st = built
    k, v = knob.split("=")
    monkeypatch.setenv(k, v)
    sm = _build(cfg, data, poses, BATCH, finalize=False)
    b2, D2, W2, _ = gpu_export_sorted(sm)
    assert np.array_equal(b2, b)
    assert np.array_equal(D2.view(np.uint32), D.view(np.uint32)) and np.array_equal(W2.view(np.uint32), W.view(np.uint32))
    st2 = sm.stats()
    assert st2["voxel_updates"] == st["voxel_updates"] and st2["total_blocks"] == st["total_blocks"]


def test_fold_inside_one_call_is_exact(lidar):
    """300 scans in one call pass the packed-accumulator limit (2^24 - 1 rays, R6/R7), so the library folds
    inside the call; the state must equal two separate calls bit for bit."""
    cfg, data, poses = lidar
    d300 = torch.cat([data, data[:100]]).contiguous()
    p300 = np.concatenate([poses, poses[:100]])
    from paper_2410_21149_b200 import Submap
    a = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    a.integrate_batch(d300, p300, cfg["sensor"])
    b = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    b.integrate_batch(d300[:150].contiguous(), p300[:150], cfg["sensor"])
    b.integrate_batch(d300[150:].contiguous(), p300[150:], cfg["sensor"])
    ea, eb = gpu_export_sorted(a), gpu_export_sorted(b)
    assert np.array_equal(ea[0], eb[0])
    assert np.array_equal(ea[1].view(np.uint32), eb[1].view(np.uint32))
    assert np.array_equal(ea[2].view(np.uint32), eb[2].view(np.uint32))
    assert a.stats()["voxel_updates"] == ea[2].astype(np.float64).sum()


def test_fullsize_frames_tsdf_parity(lidar, orc):
    cfg, data, poses = lidar
    frames = [0, 100, 199]
    sub = dict(cfg)
    sub["frames"] = {k: dict(data=data[k].cpu(), T_world_sensor=poses[k]) for k in frames}
    from paper_2410_21149_b200 import Submap
    sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    sm.integrate_batch(data[frames].contiguous(), poses[frames], cfg["sensor"])
    o, _ = oracle_build(sub, frames)
    rep = assert_tsdf_parity(gpu_export_sorted(sm), o.export())
    assert rep["observed"] > 1_000_000


def test_fullsize_esdf_sampled_brute_force(lidar, built, orc):
    cfg, _, _ = lidar
    sm, (b, D, W, E), _ = built
    g = cfg["grid"]
    rng = np.random.default_rng(0)
    l = np.arange(512)
    obs = np.argwhere(W > 0)
    unobs = np.argwhere(W == 0)
    pick = np.concatenate([obs[rng.choice(len(obs), 3000, replace=False)],
                           unobs[rng.choice(len(unobs), 300, replace=False)]])
    vox = np.stack([8 * b[pick[:, 0], 0] + pick[:, 1] % 8, 8 * b[pick[:, 0], 1] + (pick[:, 1] // 8) % 8,
                    8 * b[pick[:, 0], 2] + pick[:, 1] // 64], -1)
    d2 = orc.esdf_sample(b, D.astype(np.float64), W.astype(np.float64), g["site_threshold"], vox)
    e = E[pick[:, 0], pick[:, 1]].astype(np.float64)
    w = W[pick[:, 0], pick[:, 1]]
    dd = D[pick[:, 0], pick[:, 1]]
    assert np.isnan(e[w == 0]).all() and not np.isnan(e[w > 0]).any()
    ok = w > 0
    ref = np.where(dd < 0, -1.0, 1.0) * g["voxel_size"] * np.sqrt(d2.astype(np.float64))
    assert (d2[ok] >= 0).all()
    assert np.abs(e[ok] - ref[ok]).max() <= TOL_E
    del l


def test_fullsize_queries_sampled(lidar, built, orc):
    cfg, _, _ = lidar
    sm, (b, D, W, E), _ = built
    lo, hi = sm.aabb()
    s = cfg["grid"]["voxel_size"]
    T = sm.T_ws
    rng = np.random.default_rng(1)
    xs = rng.uniform(lo * 8 * s, (hi + 1) * 8 * s, (50000, 3))
    xw = (xs @ T[:3, :3].T + T[:3, 3]).astype(np.float32)
    dist, st = sm.query(torch.from_numpy(xw).cuda())
    dist, st = dist.cpu().numpy(), st.cpu().numpy()
    vo, so = orc.query(b, E.astype(np.float64), s, T, xw)
    assert np.array_equal(st, so)
    m = so != 2
    assert np.allclose(dist[m], vo[m], atol=1e-4, rtol=0)
    assert (so == 0).sum() > 1000


def test_fullsize_all_200_scans_parity_vs_oracle(lidar, built, orc):
    """The bench's submap state (200 scans, one launch) element by element against the oracle integrating
    all 200 scans (O1-O8; ~90 s single-threaded): block sets and observed sets bit-exact, |dD| <= 1e-4 m,
    |dW| <= 1e-3 max(1, W); then the oracle's exact EDT (O10-O12) over the GPU's exported TSDF equals the
    GPU ESDF on every voxel (stage-isolated, R4)."""
    cfg, data, poses = lidar
    sm, (b, D, W, E), st = built
    sub = dict(cfg)
    sub["frames"] = {k: dict(data=data[k].cpu(), T_world_sensor=poses[k]) for k in range(200)}
    o, _ = oracle_build(sub, range(200))
    rep = assert_tsdf_parity((b, D, W, E), o.export())
    assert rep["blocks"] == st["total_blocks"] and rep["observed"] > 5_000_000
    g = cfg["grid"]
    Eo, _ = orc.esdf(b, D.astype(np.float64), W.astype(np.float64), g["voxel_size"], g["site_threshold"])
    assert np.array_equal(np.isnan(E), np.isnan(Eo))
    fin = np.isfinite(Eo)
    assert np.abs(E[fin].astype(np.float64) - Eo[fin]).max() <= TOL_E
