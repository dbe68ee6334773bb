"""Multi-rank host logic on CPU (gloo, world_size 2): submap sharding and the packed-ESDF gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_21149_b200.parallel import gather_packed, shard_submaps


def test_lpt_sharding():
    work = [5, 1, 4, 2, 3, 3, 8]
    s = shard_submaps(work, 3)
    assert sorted(i for r in s for i in r) == list(range(len(work)))
    loads = [sum(work[i] for i in r) for r in s]
    assert max(loads) - min(loads) <= max(work)
    assert shard_submaps(work, 3) == s                      # deterministic
    assert shard_submaps([1.0] * 4, 1) == [[0, 1, 2, 3]]
    assert shard_submaps([], 2) == [[], []]


def _payload(rank, nb):
    """A cvx_pack_esdf-layout payload built in Python (header + nb records)."""
    hdr = np.zeros(256, np.uint8)
    hdr[:4] = np.frombuffer(np.uint32(0x45585643).tobytes(), np.uint8)
    hdr[4:8] = np.frombuffer(np.int32(1).tobytes(), np.uint8)
    hdr[8:16] = np.frombuffer(np.int64(nb).tobytes(), np.uint8)
    hdr[16:24] = np.frombuffer(np.float64(0.2).tobytes(), np.uint8)
    T = np.eye(4)
    T[0, 3] = rank
    hdr[24:152] = np.frombuffer(T.tobytes(), np.uint8)
    rec = np.zeros((nb, 16 + 2048), np.uint8)
    for b in range(nb):
        rec[b, :16] = np.frombuffer(np.array([rank, b, -b, b], np.int32).tobytes(), np.uint8)
        rec[b, 16:] = np.frombuffer(np.full(512, rank * 100 + b, np.float32).tobytes(), np.uint8)
    return torch.from_numpy(np.concatenate([hdr, rec.reshape(-1)]))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_21149_b200.cvx import unpack
        parts = gather_packed(_payload(rank, 3 + 2 * rank))
        res = []
        for r, p in enumerate(parts):
            d = unpack(p)
            res.append((r, d["bxyz"].shape[0], float(d["T_world_submap"][0, 3]), float(d["E"][-1, 0]),
                        d["bxyz"][:, 0].tolist()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gather_packed_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        res = out[rank]
        assert [r[1] for r in res] == [3, 5]                       # every rank sees every payload
        assert [r[2] for r in res] == [0.0, 1.0]                   # submap poses intact
        assert res[0][3] == 2.0 and res[1][3] == 104.0             # last record's E
        assert res[1][4] == [1] * 5


def _worker_esdfs(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_21149_b200.cvx import unpack
        from paper_2410_21149_b200.parallel import gather_esdfs
        mine = [_payload(10 * rank + j, 2 + j + rank) for j in range(rank + 1)]   # rank r: r + 1 payloads
        buf, offsets, counts = gather_esdfs(mine, max_per_rank=2)
        res = []
        for o in offsets:
            nb = int(np.frombuffer(buf[o + 8:o + 16].numpy().tobytes(), np.int64)[0])
            d = unpack(buf[o:o + 256 + nb * 2064])
            res.append((float(d["T_world_submap"][0, 3]), d["bxyz"].shape[0], float(d["E"][-1, 0])))
        q.put((rank, (counts, [o % 16 for o in offsets], res)))
    finally:
        dist.destroy_process_group()


def test_gather_esdfs_gloo_world2():
    """gather_esdfs: uneven payload counts per rank, one size exchange, one gather; every rank
    gets every payload at the returned offsets (16-byte aligned, as cvx_esdf_set_create needs)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_esdfs, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(0.0, 2, 1.0), (10.0, 3, 1002.0), (11.0, 4, 1103.0)]
    for rank in (0, 1):
        counts, align, res = out[rank]
        assert counts == [1, 2] and align == [0, 0, 0]
        assert res == want
