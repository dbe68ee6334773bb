"""Sharded build + gather (SURVEY §8 row e, §8c multi-GPU pin): two ranks (gloo; both on cuda:0 here —
the driver's GPU box has one device) each build the submaps longest-processing-time assigns them, pack
their ESDFs and all-gather them; every rank's gathered set equals the single-process build of all
submaps bit for bit (block sets, E), and queries through the gathered cvx_esdf_set equal each submap's
own query bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SUBMAPS = [0, 1, 2, 3, 4]
SCANS = 4


def _setup():
    import synth
    base = synth.make_config("mav", frames=[])
    frames = sorted(k for i in SUBMAPS for k in base["submaps"][i]["frames"][:SCANS])
    cfg = synth.make_config("mav", frames=frames)
    grid = dict(cfg["grid"], max_blocks=1 << 15)
    return base, cfg, grid


def _build(cfg, base, grid, i, dev):
    from paper_2410_21149_b200 import Submap
    sm = Submap(grid, base["submaps"][i]["T_world_submap"], dev.index)
    ks = base["submaps"][i]["frames"][:SCANS]
    data = torch.stack([cfg["frames"][k]["data"] for k in ks]).to(dev).contiguous()
    poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in ks])
    sm.integrate_batch(data, poses, cfg["sensor"])
    sm.finalize_esdf()
    return sm


def _sorted_records(payload):
    from paper_2410_21149_b200 import unpack
    u = unpack(payload)
    o = np.lexsort((u["bxyz"][:, 2], u["bxyz"][:, 1], u["bxyz"][:, 0]))
    return u["bxyz"][o], u["E"][o].view(np.uint32), u["T_world_submap"]


def _points(base, i, n=3000, seed=0):
    rng = np.random.default_rng(seed + i)
    T = base["submaps"][i]["T_world_submap"]
    xs = rng.uniform([-30, -30, -2], [30, 30, 6], (n, 3))
    return (xs @ T[:3, :3].T + T[:3, 3]).astype(np.float32)


def _rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_21149_b200 import EsdfSet
        from paper_2410_21149_b200.parallel import gather_esdfs, scan_work, shard_submaps
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        base, cfg, grid = _setup()
        work = [scan_work(torch.stack([cfg["frames"][k]["data"] for k in base["submaps"][i]["frames"][:SCANS]]))
                for i in SUBMAPS]
        assign = shard_submaps(work, world)
        mine = [SUBMAPS[j] for j in assign[rank]]
        packs = [_build(cfg, base, grid, i, dev).pack().cpu() for i in mine]
        buf, offsets, counts = gather_esdfs(packs, max_per_rank=max(len(a) for a in assign))
        order = [SUBMAPS[j] for a in assign for j in a]          # gathered submap ids, rank-major
        recs = {}
        for i, o in zip(order, offsets):
            nb = int(np.frombuffer(buf[o + 8:o + 16].numpy().tobytes(), np.int64)[0])
            recs[i] = _sorted_records(buf[o:o + 256 + nb * 2064])
        es = EsdfSet(buf.to(dev), offsets)
        qres = {}
        for k, i in enumerate(order):
            P = torch.from_numpy(_points(base, i)).to(dev)
            d, g, st = es.query(torch.full((P.shape[0],), k, dtype=torch.int32, device=dev), P, gradient=True)
            qres[i] = (d.cpu().numpy().view(np.uint32), g.cpu().numpy().view(np.uint32), st.cpu().numpy())
        q.put((rank, (assign, counts, recs, qres)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_build_and_gather_equal_single_process():
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(qu.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    base, cfg, grid = _setup()
    assign = out[0][0]
    assert sorted(j for a in assign for j in a) == list(range(len(SUBMAPS)))
    assert min(len(a) for a in assign) >= 1                   # both ranks build something
    for i in SUBMAPS:
        sm = _build(cfg, base, grid, i, dev)
        b, E, T = _sorted_records(sm.pack())
        P = torch.from_numpy(_points(base, i)).to(dev)
        d, g, st = sm.query_gradient(P)
        for rank in (0, 1):
            _, counts, recs, qres = out[rank]
            rb, rE, rT = recs[i]
            assert np.array_equal(rb, b) and np.array_equal(rE, E) and np.array_equal(rT, T)
            qd, qg, qs = qres[i]
            assert np.array_equal(qs, st.cpu().numpy())
            assert np.array_equal(qd, d.cpu().numpy().view(np.uint32))
            assert np.array_equal(qg, g.cpu().numpy().view(np.uint32))
            assert (qs == 0).sum() > 100
