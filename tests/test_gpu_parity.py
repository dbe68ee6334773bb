"""GPU parity: libcvx (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): block sets and observed sets bit-exact; |dD| <= 1e-4 m,
|dW| <= 1e-3 * max(1, W); |dE| <= 1e-4 m with identical NaN / +inf patterns; query values within
1e-4 m and identical statuses.
"""
import math

import numpy as np
import pytest
import torch

import synth
from helpers import (TOL_E, assert_esdf_parity, assert_tsdf_parity, gpu_build, gpu_export_sorted,
                     oracle_build, sort_blocks)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    return synth.make_config("tiny")


def _cum_stats(stats_list):
    keys = ("rays_in", "rays_used", "skipped_invalid", "skipped_range", "skipped_domain", "voxel_updates")
    return {k: sum(s[k] for s in stats_list) for k in keys}


def test_tiny_tsdf_parity_and_counts(tiny, orc):
    frames = list(range(10))
    sm, st = gpu_build(tiny, frames, finalize=False)
    o = orc.OracleSubmap(tiny["grid"], tiny["submaps"][0]["T_world_submap"])
    ost = [o.integrate(tiny["frames"][k]["data"].numpy(), tiny["frames"][k]["T_world_sensor"], tiny["sensor"])
           for k in frames]
    rep = assert_tsdf_parity(gpu_export_sorted(sm), o.export())
    cum = _cum_stats(ost)
    for k, v in cum.items():
        assert st[k] == v, (k, st[k], v)
    assert st["total_blocks"] == o.num_blocks() == rep["blocks"]
    # COUNT closed form == what the walk deposits: sum of W over voxels (constant weights)
    _, _, W, _ = gpu_export_sorted(sm)
    assert W.astype(np.float64).sum() == st["voxel_updates"]


def test_batch_equals_sequential_bitexact_and_deterministic(tiny):
    frames = list(range(10))
    a, _ = gpu_build(tiny, frames, batch=False, finalize=False)
    b, _ = gpu_build(tiny, frames, batch=True, finalize=False)
    c, _ = gpu_build(tiny, list(reversed(frames)), batch=True, finalize=False)
    ea, eb, ec = gpu_export_sorted(a), gpu_export_sorted(b), gpu_export_sorted(c)
    for x, y in ((ea, eb), (ea, ec)):
        assert np.array_equal(x[0], y[0])
        assert np.array_equal(x[1].view(np.uint32), y[1].view(np.uint32))   # D bitwise
        assert np.array_equal(x[2].view(np.uint32), y[2].view(np.uint32))   # W bitwise


@pytest.mark.parametrize("weighting,carve", [(1, 1), (0, 0), (1, 0)])
def test_tiny_modes_parity(tiny, orc, weighting, carve):
    g = dict(tiny["grid"], weighting=weighting, carve=carve)
    frames = [0, 3, 7]
    sm, _ = gpu_build(tiny, frames, grid=g, finalize=False)
    o, _ = oracle_build(tiny, frames, grid=g)
    assert_tsdf_parity(gpu_export_sorted(sm), o.export())


def test_lidar_subset_parity(orc):
    cfg = synth.make_config("lidar", frames=[0, 60])
    sm, st = gpu_build(cfg, [0, 60], finalize=False)
    o, _ = oracle_build(cfg, [0, 60])
    rep = assert_tsdf_parity(gpu_export_sorted(sm), o.export())
    assert rep["blocks"] > 5000


@pytest.mark.parametrize("isub,min_blocks", [(2, 5000), (7, 100)])   # outdoors; inside the building
def test_mav_submap_parity(orc, isub, min_blocks):
    """BASELINE.json configs[3]: one MAV submap (its own pose, the disaster-site scene) over 4 scans with
    range weighting — TSDF parity and the stage-isolated exact ESDF on every voxel."""
    base = synth.make_config("mav", frames=[])
    sub = base["submaps"][isub]
    ks = sub["frames"][:40:10]
    cfg = synth.make_config("mav", frames=ks)
    g = dict(cfg["grid"], weighting=1, max_blocks=1 << 16)
    sm, _ = gpu_build(cfg, ks, grid=g, T_ws=sub["T_world_submap"], batch=True)
    o, _ = oracle_build(cfg, ks, grid=g, T_ws=sub["T_world_submap"])
    b, D, W, E = gpu_export_sorted(sm)
    rep = assert_tsdf_parity((b, D, W, E), o.export())
    assert rep["blocks"] > min_blocks
    Eo, _ = orc.esdf(b, D.astype(np.float64), W.astype(np.float64), g["voxel_size"], g["site_threshold"])
    assert_esdf_parity(E, Eo, W > 0)


def test_rgbd_subset_parity(orc):
    cfg = synth.make_config("rgbd", frames=[0, 37])
    sm, _ = gpu_build(cfg, [0, 37], grid=dict(cfg["grid"], weighting=1), finalize=False)
    o, _ = oracle_build(cfg, [0, 37], grid=dict(cfg["grid"], weighting=1))
    assert_tsdf_parity(gpu_export_sorted(sm), o.export())


def test_pose_composition_nontrivial_submap_pose(tiny, orc):
    T = synth.pose(synth.rot_zyx(0.7, 0.1, -0.2), [0.3, -1.7, 0.25])
    sm, _ = gpu_build(tiny, [0, 5, 9], T_ws=T, finalize=False)
    o, _ = oracle_build(tiny, [0, 5, 9], T_ws=T)
    assert_tsdf_parity(gpu_export_sorted(sm), o.export())


# ------------------------------------------------------------------------------------------ ESDF
def test_tiny_esdf_stage_isolated_and_end_to_end(tiny, orc):
    frames = list(range(10))
    sm, _ = gpu_build(tiny, frames)
    b, D, W, E = gpu_export_sorted(sm)
    g = tiny["grid"]
    # stage-isolated: the oracle EDT on the GPU's exported TSDF (identical site sets)
    Eo, _ = orc.esdf(b, D.astype(np.float64), W.astype(np.float64), g["voxel_size"], g["site_threshold"])
    assert_esdf_parity(E, Eo, W > 0)
    # brute force agrees too (tiny config: O(|O| |S|))
    Eb, _ = orc.esdf(b, D.astype(np.float64), W.astype(np.float64), g["voxel_size"], g["site_threshold"], brute=True)
    assert_esdf_parity(E, Eb, W > 0)
    # end-to-end: oracle TSDF -> oracle ESDF; voxels beyond tolerance come only from site-threshold ties
    o, _ = oracle_build(tiny, frames)
    bo, Do, Wo = o.export()
    Eoe, _ = orc.esdf(bo, Do, Wo, g["voxel_size"], g["site_threshold"])
    fin = np.isfinite(Eoe)
    bad = (np.abs(E.astype(np.float64) - Eoe)[fin] > TOL_E).sum()
    assert bad <= 0.001 * fin.sum(), bad


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_esdf_import_random_tsdf(orc, seed):
    """Stage-isolated ESDF on imported random TSDFs: holes, ragged AABB, negative coordinates."""
    from paper_2410_21149_b200 import Submap
    rng = np.random.default_rng(seed)
    blocks = [(x, y, z) for x in range(-2, 3) for y in range(-1, 3) for z in range(-1, 2) if rng.random() < 0.7]
    b = np.array(blocks, np.int32)
    nb = len(b)
    W = ((rng.random((nb, 512)) < 0.85) * rng.uniform(0.5, 4, (nb, 512))).astype(np.float32)
    D = (rng.uniform(-0.3, 0.3, (nb, 512)) * (W > 0)).astype(np.float32)
    grid = dict(voxel_size=0.1, truncation=0.3, site_threshold=0.01, max_blocks=4096)
    sm = Submap(grid)
    dev = torch.device("cuda", 0)
    sm.import_tsdf(torch.from_numpy(b).to(dev), torch.from_numpy(D).to(dev), torch.from_numpy(W).to(dev))
    sm.finalize_esdf()
    bg, Dg, Wg, Eg = gpu_export_sorted(sm)
    bs, Ds, Ws = sort_blocks(b, D, W)
    assert np.array_equal(bg, bs)
    Eo, _ = orc.esdf(bg, Dg.astype(np.float64), Wg.astype(np.float64), 0.1, 0.01)
    assert_esdf_parity(Eg, Eo, Wg > 0)


@pytest.mark.parametrize("seed,p_site", [(0, 2e-4), (1, 3e-3), (2, 0.05)])
def test_esdf_long_lines_sparse_sites(orc, seed, p_site):
    """Lines longer than one TMA box (y: 360, z: 320 voxels) with sparse and dense site patterns, holes and
    a ragged block set: exercises the banded envelopes, empty bands and every merge level of passes y / z."""
    from paper_2410_21149_b200 import Submap
    rng = np.random.default_rng(50 + seed)
    blocks = [(x, y, z) for x in range(0, 3) for y in range(-20, 25) for z in range(-15, 25) if rng.random() < 0.6]
    b = np.array(blocks, np.int32)
    nb = len(b)
    W = ((rng.random((nb, 512)) < 0.9) * rng.uniform(0.5, 4, (nb, 512))).astype(np.float32)
    D = rng.uniform(0.02, 0.3, (nb, 512)) * np.where(rng.random((nb, 512)) < 0.5, -1, 1)
    site = rng.random((nb, 512)) < p_site
    D = (np.where(site, rng.uniform(-0.01, 0.01, (nb, 512)), D) * (W > 0)).astype(np.float32)
    grid = dict(voxel_size=0.1, truncation=0.3, site_threshold=0.01, max_blocks=nb + 16)
    sm = Submap(grid)
    dev = torch.device("cuda", 0)
    sm.import_tsdf(torch.from_numpy(b).to(dev), torch.from_numpy(D).to(dev), torch.from_numpy(W).to(dev))
    sm.finalize_esdf()
    bg, Dg, Wg, Eg = gpu_export_sorted(sm)
    Eo, _ = orc.esdf(bg, Dg.astype(np.float64), Wg.astype(np.float64), 0.1, 0.01)
    assert_esdf_parity(Eg, Eo, Wg > 0)


def test_esdf_no_sites_and_single_site(orc):
    from paper_2410_21149_b200 import Submap
    dev = torch.device("cuda", 0)
    b = torch.tensor([[0, 0, 0], [3, -1, 2]], dtype=torch.int32, device=dev)
    W = torch.ones((2, 512), device=dev)
    W[1, :7] = 0
    D = torch.full((2, 512), 0.25, device=dev)
    sm = Submap(dict(voxel_size=0.05, truncation=0.3, site_threshold=0.05, max_blocks=64))
    sm.import_tsdf(b, D, W)
    sm.finalize_esdf()
    _, _, Wg, Eg = gpu_export_sorted(sm)
    assert np.isposinf(Eg[Wg > 0]).all() and np.isnan(Eg[Wg == 0]).all()
    D2 = D.clone()
    D2[1, 100] = 0.0
    D2[0, :] = -0.25
    sm2 = Submap(dict(voxel_size=0.05, truncation=0.3, site_threshold=0.05, max_blocks=64))
    sm2.import_tsdf(b, D2, W)
    sm2.finalize_esdf()
    bg, Dg, Wg, Eg = gpu_export_sorted(sm2)
    Eo, _ = orc.esdf(bg, Dg.astype(np.float64), Wg.astype(np.float64), 0.05, 0.05, brute=True)
    assert_esdf_parity(Eg, Eo, Wg > 0)
    assert (Eg[bg[:, 0] == 0] < 0).all()


# ------------------------------------------------------------------------------------------ query
def test_query_parity(tiny, orc):
    T = synth.pose(synth.rot_zyx(0.3), [0.5, 0.25, -0.1])
    sm, _ = gpu_build(tiny, list(range(10)), T_ws=T)
    b, D, W, E = gpu_export_sorted(sm)
    lo, hi = sm.aabb()
    rng = np.random.default_rng(0)
    s = tiny["grid"]["voxel_size"]
    xs = rng.uniform(lo * 8 * s - 0.5, (hi + 1) * 8 * s + 0.5, (20000, 3))
    xw = (xs @ T[:3, :3].T + T[:3, 3]).astype(np.float32)
    dist, st = sm.query(torch.from_numpy(xw).cuda())
    dist, st = dist.cpu().numpy(), st.cpu().numpy()
    vo, so = orc.query(b, E.astype(np.float64), s, T, xw)
    assert np.array_equal(st, so)
    ok = so != 2
    assert np.allclose(dist[ok], vo[ok], atol=1e-4, rtol=0)
    assert np.isnan(dist[~ok]).all()
    assert (so == 0).sum() > 300 and (so == 1).sum() > 10 and (so == 2).sum() > 100


# ------------------------------------------------------------------------------------------ edges
def test_edge_cases_and_errors(tiny):
    from paper_2410_21149_b200 import CvxError, Submap
    dev = torch.device("cuda", 0)
    sm = Submap(tiny["grid"])
    # empty frame: no-op; all-invalid frame counted
    st = sm.integrate(torch.zeros((0, 3), device=dev), np.eye(4), dict(kind=0, min_range=0.1, max_range=5.0), stats=True)
    assert st["rays_in"] == 0 and st["total_blocks"] == 0
    bad = torch.full((33, 3), float("nan"), device=dev)
    st = sm.integrate(bad, np.eye(4), dict(kind=0, min_range=0.1, max_range=5.0), stats=True)
    assert st["skipped_invalid"] == 33 and st["total_blocks"] == 0
    with pytest.raises(CvxError) as ei:
        sm.query(torch.zeros((4, 3), device=dev))
    assert ei.value.code == -4                 # query before finalize
    sm.finalize_esdf()                          # empty submap finalizes
    with pytest.raises(CvxError) as ei:
        sm.integrate(torch.zeros((1, 3), device=dev), np.eye(4), dict(kind=0))
    assert ei.value.code == -4                 # integrate after finalize
    d, s = sm.query(torch.zeros((4, 3), device=dev))
    assert (s.cpu().numpy() == 2).all()
    # capacity overflow -> CVX_E_CAPACITY at the next synchronising call
    small = Submap(dict(tiny["grid"], max_blocks=4))
    small.integrate(tiny["frames"][0]["data"].to(dev), tiny["frames"][0]["T_world_sensor"], tiny["sensor"])
    with pytest.raises(CvxError) as ei:
        small.finalize_esdf()
    assert ei.value.code == -3
    # ray beyond the 21-bit key domain -> CVX_E_RANGE, ray skipped and counted
    far = Submap(dict(voxel_size=0.001, truncation=0.003, max_blocks=1024))
    pts = torch.tensor([[1.0, 0.0, 0.0], [9000.0, 0.0, 0.0]], device=dev)
    with pytest.raises(CvxError) as ei:
        far.integrate(pts, np.eye(4), dict(kind=0, min_range=0.0, max_range=1e6), stats=True)
    assert ei.value.code == -6
    # invalid arguments are rejected synchronously
    with pytest.raises(CvxError):
        Submap(dict(tiny["grid"], block_side=16))
    T = np.eye(4)
    T[0, 0] = 2.0
    with pytest.raises(CvxError):
        Submap(tiny["grid"], T)


def test_reset_and_pack_roundtrip(tiny):
    from paper_2410_21149_b200 import Submap, unpack
    sm, _ = gpu_build(tiny, [0, 1, 2])
    b, D, W, E = gpu_export_sorted(sm)
    payload = unpack(sm.pack())
    pb, pE = sort_blocks(payload["bxyz"], payload["E"])
    assert np.array_equal(pb, b) and np.array_equal(pE.view(np.uint32), E.view(np.uint32))
    assert np.allclose(payload["T_world_submap"], sm.T_ws)
    # reset -> identical rebuild
    sm.reset()
    assert sm.block_count() == 0
    dev = torch.device("cuda", 0)
    for k in (0, 1, 2):
        sm.integrate(tiny["frames"][k]["data"].to(dev), tiny["frames"][k]["T_world_sensor"], tiny["sensor"])
    sm.finalize_esdf()
    b2, D2, W2, E2 = gpu_export_sorted(sm)
    assert np.array_equal(b2, b) and np.array_equal(D2.view(np.uint32), D.view(np.uint32))
    assert np.array_equal(E2.view(np.uint32), E.view(np.uint32))


def test_wide_and_narrow_dda_paths_agree(tiny, orc):
    """A sensor max range beyond 4096 voxels selects the 64-bit crossing-order path of the walk; the
    32-bit path (default) and the 64-bit path must give bit-identical TSDFs and match the oracle."""
    frames = [0, 4, 8]
    narrow, _ = gpu_build(tiny, frames, finalize=False)
    wide_cfg = dict(tiny, sensor=dict(tiny["sensor"], max_range=1.0e6))
    wide, _ = gpu_build(wide_cfg, frames, finalize=False)
    a, b = gpu_export_sorted(narrow), gpu_export_sorted(wide)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    assert np.array_equal(a[2].view(np.uint32), b[2].view(np.uint32))
    o, _ = oracle_build(wide_cfg, frames)
    assert_tsdf_parity(b, o.export())


def test_host_frames_equal_device_frames(tiny):
    """cvx_integrate_batch_host (library-side overlapped H2D copies) == cvx_integrate_batch, bit for bit."""
    from paper_2410_21149_b200 import Submap
    frames = list(range(10))
    a, _ = gpu_build(tiny, frames, batch=True, finalize=False)
    b = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    host = torch.stack([tiny["frames"][k]["data"] for k in frames]).contiguous().pin_memory()
    poses = np.stack([tiny["frames"][k]["T_world_sensor"] for k in frames])
    b.integrate_batch_host(host, poses, tiny["sensor"])
    ea, eb = gpu_export_sorted(a), gpu_export_sorted(b)
    assert np.array_equal(ea[0], eb[0])
    assert np.array_equal(ea[1].view(np.uint32), eb[1].view(np.uint32))
    assert np.array_equal(ea[2].view(np.uint32), eb[2].view(np.uint32))


def test_reset_with_new_pose_matches_fresh_submap(tiny):
    """cvx_reset_submap + cvx_set_submap_pose == a freshly created submap with that pose (bitwise)."""
    from paper_2410_21149_b200 import Submap
    T2 = synth.pose(synth.rot_zyx(-0.4), [0.2, 0.1, -0.3])
    a, _ = gpu_build(tiny, [0, 1], finalize=False)
    a.reset(T2)
    dev = torch.device("cuda", 0)
    for k in (2, 3):
        a.integrate(tiny["frames"][k]["data"].to(dev), tiny["frames"][k]["T_world_sensor"], tiny["sensor"])
    b, _ = gpu_build(tiny, [2, 3], T_ws=T2, finalize=False)
    ea, eb = gpu_export_sorted(a), gpu_export_sorted(b)
    assert np.array_equal(ea[0], eb[0]) and np.array_equal(ea[1].view(np.uint32), eb[1].view(np.uint32))


def test_block_count_trigger_matches_frame_by_frame(tiny):
    """cvx_integrate_until (P:L115 block-count submap trigger, checked on the device) takes exactly the
    frames a host loop would (integrate one frame, read the block count, stop at the threshold), with a
    bit-identical TSDF."""
    from paper_2410_21149_b200 import Submap
    dev = torch.device("cuda", 0)
    frames = list(range(10))
    data = torch.stack([tiny["frames"][k]["data"] for k in frames]).to(dev).contiguous()
    poses = np.stack([tiny["frames"][k]["T_world_sensor"] for k in frames])
    ref = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    counts = []
    for k in frames:
        ref.integrate(data[k].contiguous(), poses[k], tiny["sensor"])
        counts.append(ref.block_count())
    thr = counts[4] if counts[4] > counts[3] else counts[4] + 1
    expect = next((i + 1 for i, c in enumerate(counts) if c >= thr), len(frames))
    a = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    took = a.integrate_until(data, poses, tiny["sensor"], thr)
    assert took == expect
    b = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    b.integrate_batch(data[:took].contiguous(), poses[:took], tiny["sensor"])
    ea, eb = gpu_export_sorted(a), gpu_export_sorted(b)
    assert np.array_equal(ea[0], eb[0]) and np.array_equal(ea[1].view(np.uint32), eb[1].view(np.uint32))
    assert a.stats()["rays_in"] == took * data[0].numel()
    # threshold never reached: every frame is taken
    c = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    assert c.integrate_until(data, poses, tiny["sensor"], tiny["grid"]["max_blocks"]) == len(frames)


@pytest.mark.parametrize("knob", ["CVX_FUSE_ALLOC=1", "CVX_BW3=1", "CVX_BW2=0", "CVX_WALK_CW=0", "CVX_LIST_CAP=2000",
                                  "CVX_DENSE=0", "CVX_DENSE_BLOCKS=4"])
def test_walk_variants_bitexact(tiny, orc, monkeypatch, knob):
    """The tuning variants of the integrate path (ALLOCATE fused into the walk, the first block walk,
    the general walk kernel; a slot-list buffer capped so most rays find their blocks by hash lookup in
    the walk; the slot-list path instead of the dense window (R19), chosen on the host or — with a window
    buffer too small for any launch's box — by the device-side fallback) read at submap creation: each must give the default path's TSDF bit for bit (R1 exact
    sums) and match the oracle."""
    frames = [0, 3, 6, 9]
    ref, _ = gpu_build(tiny, frames, batch=True, finalize=False)
    for kv in knob.split(","):
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    var, _ = gpu_build(tiny, frames, batch=True, finalize=False)
    a, b = gpu_export_sorted(ref), gpu_export_sorted(var)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    assert np.array_equal(a[2].view(np.uint32), b[2].view(np.uint32))
    o, _ = oracle_build(tiny, frames)
    assert_tsdf_parity(b, o.export())


def test_host_frames_two_submaps_in_flight(tiny):
    """The bench's schedule with host frames: two submaps on two streams; after checking submap k's round
    r, its round r + 1 (other frames) is issued while the other submap's round r may still run.  The
    host-frame copies are not ordered after earlier work on the caller's stream (they wait only for the
    prepare that last read their staging buffer), so this checks that the early copies never feed a
    prepare stale or foreign data: every round must equal a device-resident call bit for bit."""
    from paper_2410_21149_b200 import Submap
    R = 4
    sets = []
    for r in range(R):
        idx = [(k + 3 * r) % 10 for k in range(240 - 20 * r)]
        dev = torch.stack([tiny["frames"][k]["data"] for k in idx]).contiguous().cuda()
        poses = np.stack([tiny["frames"][k]["T_world_sensor"] for k in idx])
        ref = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
        ref.integrate_batch(dev, poses, tiny["sensor"])
        sets.append((dev.cpu().pin_memory(), poses, gpu_export_sorted(ref)))
    subs = [Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0) for _ in range(2)]
    streams = [torch.cuda.current_stream(), torch.cuda.Stream()]

    def issue(k, r):
        with torch.cuda.stream(streams[k]):
            subs[k].reset()
            subs[k].integrate_batch_host(sets[r][0], sets[r][1], tiny["sensor"])

    issue(0, 0)
    issue(1, 0)
    for r in range(R):
        for k in (0, 1):
            with torch.cuda.stream(streams[k]):   # stream-local sync: the other submap keeps running
                b, D, W, E = subs[k].export(with_esdf=True)
                streams[k].synchronize()
            e = sort_blocks(b.cpu().numpy(), D.cpu().numpy(), W.cpu().numpy(), E.cpu().numpy())
            er = sets[r][2]
            assert np.array_equal(er[0], e[0]), (r, k)
            assert np.array_equal(er[1].view(np.uint32), e[1].view(np.uint32)), (r, k)
            assert np.array_equal(er[2].view(np.uint32), e[2].view(np.uint32)), (r, k)
            if r + 1 < R:
                issue(k, r + 1)


def test_host_frames_many_launches_and_calls(tiny):
    """Host frames over several walk launches (300 frames > kMaxBatch = 200 per launch) and several calls
    of uneven size: the copy stream refills the two staging buffers while earlier launches are still
    being ingested; the TSDF must equal one device-resident call bit for bit."""
    from paper_2410_21149_b200 import Submap
    idx = [k % 10 for k in range(300)]
    dev_frames = torch.stack([tiny["frames"][k]["data"] for k in idx]).contiguous()
    poses = np.stack([tiny["frames"][k]["T_world_sensor"] for k in idx])
    a = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    a.integrate_batch(dev_frames.cuda(), poses, tiny["sensor"])
    b = Submap(tiny["grid"], tiny["submaps"][0]["T_world_submap"], 0)
    host = dev_frames.pin_memory()
    for lo, hi in ((0, 100), (100, 250), (250, 300)):
        b.integrate_batch_host(host[lo:hi], poses[lo:hi], tiny["sensor"])
    ea, eb = gpu_export_sorted(a), gpu_export_sorted(b)
    assert np.array_equal(ea[0], eb[0])
    assert np.array_equal(ea[1].view(np.uint32), eb[1].view(np.uint32))
    assert np.array_equal(ea[2].view(np.uint32), eb[2].view(np.uint32))
    assert a.stats()["rays_used"] == b.stats()["rays_used"] > 0


@pytest.mark.parametrize("name,frames", [("tiny", list(range(10))), ("lidar", [0, 20, 40, 60, 80, 100])])
def test_block_count_trigger_matches_oracle(orc, name, frames):
    """cvx_integrate_until (the submap ends once it holds block_threshold blocks) against the
    ORACLE's per-frame block counts (orc_num_blocks after each frame, O7): the frame at which the oracle's
    block set first reaches the threshold is the last one the GPU takes, and the GPU submap after the call
    equals the oracle's submap of those frames (block sets bit-exact, TSDF within tolerance)."""
    from paper_2410_21149_b200 import Submap
    cfg = synth.make_config(name, frames=frames)
    o = orc.OracleSubmap(cfg["grid"], cfg["submaps"][0]["T_world_submap"])
    counts = []
    for k in frames:
        o.integrate(cfg["frames"][k]["data"].numpy(), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
        counts.append(o.num_blocks())
    dev = torch.device("cuda", 0)
    data = torch.stack([cfg["frames"][k]["data"] for k in frames]).to(dev).contiguous()
    poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in frames])
    for j in range(1, len(frames)):
        if counts[j] == counts[j - 1]:
            continue
        for thr in (counts[j], counts[j - 1] + 1):          # reached exactly / just past the previous count
            expect = next(i + 1 for i, c in enumerate(counts) if c >= thr)
            sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
            took = sm.integrate_until(data, poses, cfg["sensor"], thr)
            assert took == expect, (thr, took, expect, counts)
            assert sm.block_count() == counts[took - 1]
        if j == len(frames) // 2:
            ref, _ = oracle_build(cfg, frames[:took])
            assert_tsdf_parity(gpu_export_sorted(sm), ref.export())
    sm = Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0)
    assert sm.integrate_until(data, poses, cfg["sensor"], counts[-1] + 1) == len(frames)


@pytest.mark.parametrize("which", ["lidar", "mav"])
def test_split_line_pass_equals_default(orc, monkeypatch, which):
    """ESDF pass y with two threads per line (CVX_EDT_SPLIT=1: forward sweeps of the two halves, the second
    half's stack merged onto the first's, R20) gives the default kernel's ESDF bit for bit, and the
    stage-isolated oracle EDT."""
    if which == "lidar":
        cfg = synth.make_config("lidar", frames=[0, 60])
        ks, g, T = [0, 60], cfg["grid"], None
    else:
        base = synth.make_config("mav", frames=[])
        sub = base["submaps"][2]
        ks = sub["frames"][:40:10]
        cfg = synth.make_config("mav", frames=ks)
        g, T = dict(cfg["grid"], max_blocks=1 << 16), sub["T_world_submap"]
    sm, _ = gpu_build(cfg, ks, grid=g, T_ws=T, batch=True)
    a = gpu_export_sorted(sm)
    monkeypatch.setenv("CVX_EDT_SPLIT", "1")
    sm2, _ = gpu_build(cfg, ks, grid=g, T_ws=T, batch=True)
    b = gpu_export_sorted(sm2)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[3].view(np.uint32), b[3].view(np.uint32))
    Eo, _ = orc.esdf(b[0], b[1].astype(np.float64), b[2].astype(np.float64), g["voxel_size"], g["site_threshold"])
    assert_esdf_parity(b[3], Eo, b[2] > 0)
