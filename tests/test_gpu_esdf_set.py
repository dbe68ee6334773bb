"""Gathered submap ESDFs (SURVEY §8 rows e / f4): cvx_esdf_set over cvx_pack_esdf payloads,
batched value + gradient look-ups across submaps, each in its own frame — against the oracle's O13 query
of each submap and against the submap's own query (same arithmetic: bit-identical)."""
import numpy as np
import pytest
import torch

import synth
from helpers import gpu_build

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def three():
    cfg = synth.make_config("tiny")
    poses = [synth.pose(synth.rot_zyx(0.3, 0.05, 0.0), [0.5, 0.25, -0.1]),
             synth.pose(synth.rot_zyx(-1.1), [-40.0, 13.0, 2.0]),
             np.eye(4)]
    frames = [[0, 1, 2, 3], [3, 4, 5, 6], [6, 7, 8, 9]]
    subs = [gpu_build(cfg, fr, T_ws=T)[0] for fr, T in zip(frames, poses)]
    return cfg, subs


def test_set_matches_oracle_and_own_query(three, orc):
    from paper_2410_21149_b200 import EsdfSet, unpack
    cfg, subs = three
    s = cfg["grid"]["voxel_size"]
    packs = [sm.pack() for sm in subs]
    # concatenate with a gap (as an all-gather with padding would) at 16-byte aligned offsets
    offsets, chunks, o = [], [], 0
    for p in packs:
        offsets.append(o)
        pad = (-p.numel()) % 16 + 48
        chunks += [p, torch.zeros(pad, dtype=torch.uint8, device=p.device)]
        o += p.numel() + pad
    buf = torch.cat(chunks).contiguous()
    es = EsdfSet(buf, offsets)
    rng = np.random.default_rng(3)
    pts, idx = [], []
    for k, sm in enumerate(subs):
        lo, hi = sm.aabb()
        xs = rng.uniform(lo * 8 * s - 0.3, (hi + 1) * 8 * s + 0.3, (6000, 3))
        pts.append(xs @ sm.T_ws[:3, :3].T + sm.T_ws[:3, 3])
        idx.append(np.full(6000, k))
    pts.append(rng.uniform(-1, 1, (200, 3)))
    idx.append(rng.choice([-1, 3, 1000], 200))                  # no such submap -> UNKNOWN
    P = np.concatenate(pts).astype(np.float32)
    I = np.concatenate(idx).astype(np.int32)
    perm = rng.permutation(len(I))                              # submaps interleaved in one batch
    P, I = P[perm], I[perm]
    d, g, st = es.query(torch.from_numpy(I).cuda(), torch.from_numpy(P).cuda(), gradient=True)
    d, g, st = d.cpu().numpy(), g.cpu().numpy(), st.cpu().numpy()
    assert (st[(I < 0) | (I >= 3)] == 2).all()
    for k, sm in enumerate(subs):
        sel = I == k
        u = unpack(packs[k])
        vo, so, go = orc.query(u["bxyz"], u["E"].astype(np.float64), u["voxel_size"], u["T_world_submap"], P[sel],
                               gradient=True)
        assert np.array_equal(st[sel], so)
        ok = so != 2
        assert (so == 0).sum() > 100
        assert np.allclose(d[sel][ok], vo[ok], atol=1e-4, rtol=0)
        fin = (so == 0) & np.isfinite(go).all(1)
        assert np.allclose(g[sel][fin], go[fin], atol=1e-4, rtol=1e-5)
        d1, g1, s1 = sm.query_gradient(torch.from_numpy(P[sel]).cuda())
        assert np.array_equal(s1.cpu().numpy(), st[sel])
        assert np.array_equal(d1.cpu().numpy().view(np.uint32), d[sel].view(np.uint32))
        assert np.array_equal(g1.cpu().numpy().view(np.uint32), g[sel].view(np.uint32))
    es.close()


def test_set_rejects_bad_payloads(three):
    from paper_2410_21149_b200 import CvxError, EsdfSet
    cfg, subs = three
    p = subs[0].pack().clone()
    with pytest.raises(CvxError):
        EsdfSet(p, [8])                                         # misaligned offset
    bad = p.clone()
    bad[0] = 0                                                  # broken magic
    with pytest.raises(CvxError):
        EsdfSet(bad, [0])
    dup = torch.cat([p, p[256:256 + 2064]])                     # one block listed twice
    dup[8:16] = torch.from_numpy(np.frombuffer(np.int64(int(np.frombuffer(p[8:16].cpu().numpy().tobytes(), np.int64)[0]) + 1).tobytes(), np.uint8).copy()).cuda()
    with pytest.raises(CvxError):
        EsdfSet(dup.contiguous(), [0])
