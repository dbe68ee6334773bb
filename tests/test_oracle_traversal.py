"""Pins of the oracle's ray extent, quantisation and traversal.

None of these re-types the oracle's walk: the references are the SPEC examples, the closed-form
count, an exact rational brute force over candidate voxels, and explicit tie cases.
"""
import math
from fractions import Fraction

import numpy as np
import pytest


def test_axis_aligned_example(orc):
    # origin (0,0,0) to (0.35,0,0), voxel 0.1, truncation 0 -> x-indices 0..3
    v = orc.ray_voxels([0, 0, 0], [0.35, 0, 0], 0.1, 0.0)
    assert v[:, 0].tolist() == [0, 1, 2, 3]
    assert (v[:, 1:] == 0).all()


def test_truncation_extension_example(orc):
    # endpoint inside the origin voxel, truncation 0.4 -> 1 + ceil(0.4/0.1) voxels
    v = orc.ray_voxels([0.05, 0.05, 0.05], [0.07, 0.05, 0.05], 0.1, 0.4)
    assert len(v) == 1 + math.ceil(0.4 / 0.1)
    assert v[:, 0].tolist() == [0, 1, 2, 3, 4]


def _exact_voxels(A, B):
    """Exact brute force: voxels whose box meets the fixed-point segment A->B with positive length,
    plus voxel(A) and voxel(B).  A, B are integer fixed-point coordinates (F = 16)."""
    one = 1 << 16
    va = [a >> 16 for a in A]
    vb = [b >> 16 for b in B]
    lo = [min(x, y) for x, y in zip(va, vb)]
    hi = [max(x, y) for x, y in zip(va, vb)]
    out = {tuple(va), tuple(vb)}
    for x in range(lo[0], hi[0] + 1):
        for y in range(lo[1], hi[1] + 1):
            for z in range(lo[2], hi[2] + 1):
                t0, t1 = Fraction(0), Fraction(1)
                for i, c in enumerate((x, y, z)):
                    d = B[i] - A[i]
                    if d == 0:
                        if not (c * one <= A[i] < (c + 1) * one):
                            t0, t1 = Fraction(1), Fraction(0)
                        continue
                    ta = Fraction(c * one - A[i], d)
                    tb = Fraction((c + 1) * one - A[i], d)
                    t0, t1 = max(t0, min(ta, tb)), min(t1, max(ta, tb))
                if t1 > t0:
                    out.add((x, y, z))
    return out


@pytest.mark.parametrize("seed", range(4))
def test_random_rays_vs_exact_brute_force(orc, seed):
    # s = 0.25 and coordinates on a 2^-20 grid: x/s*2^16 is exact, so the fixed-point endpoints are
    # known exactly without re-typing the quantisation; tau = 0 so the extent is exactly p.
    rng = np.random.default_rng(seed)
    s = 0.25
    for _ in range(60):
        o = rng.integers(-3 << 20, 3 << 20, 3) / float(1 << 20)
        p = o + rng.integers(-4 << 20, 4 << 20, 3) / float(1 << 20)
        v = orc.ray_voxels(o, p, s, 0.0)
        A = [int(round(x / s * 65536)) for x in o]
        B = [int(round(x / s * 65536)) for x in p]
        ref = _exact_voxels(A, B)
        got = [tuple(r) for r in v.tolist()]
        # closed-form count (a2): 1 + sum |dv|
        assert len(got) == 1 + sum(abs((b >> 16) - (a >> 16)) for a, b in zip(A, B))
        # no duplicates, exact set, 6-connected, starts at voxel(A), ends at voxel(B)
        assert len(set(got)) == len(got)
        assert set(got) == ref
        assert got[0] == tuple(a >> 16 for a in A) and got[-1] == tuple(b >> 16 for b in B)
        steps = np.abs(np.diff(np.array(got), axis=0)).sum(1)
        assert (steps == 1).all()


def test_dense_sampling_subset(orc):
    # a dense sampler at 1/100 voxel only ever finds voxels the walk visits.
    rng = np.random.default_rng(7)
    s, tau = 0.1, 0.3
    for _ in range(200):
        o = rng.uniform(-2, 2, 3)
        p = o + rng.normal(0, 1.5, 3)
        v = orc.ray_voxels(o, p, s, tau)
        d = p - o
        L = np.linalg.norm(d)
        e = p + tau * d / L
        n = int(np.ceil(np.linalg.norm(e - o) / s * 100)) + 1
        t = np.linspace(0.0, 1.0, n)[1:-1]
        pts = o[None] + t[:, None] * (e - o)[None]
        sampled = {tuple(r) for r in np.floor(pts / s).astype(np.int64).tolist()}
        walk = {tuple(r) for r in v.tolist()}
        assert sampled <= walk
        assert len(walk) - len(sampled) <= 4  # only corner clips thinner than the sampling step may be missed


def test_tie_breaks_x_before_y_before_z(orc):
    # ray through the exact edge between voxels: the walk steps x first (O4, Q8)
    v = orc.ray_voxels([0.5, 0.5, 0.5], [2.5, 2.5, 0.5], 1.0, 0.0)
    assert [tuple(r) for r in v.tolist()] == [(0, 0, 0), (1, 0, 0), (1, 1, 0), (2, 1, 0), (2, 2, 0)]
    v = orc.ray_voxels([0.5, 0.5, 0.5], [0.5, 1.5, 1.5], 1.0, 0.0)
    assert [tuple(r) for r in v.tolist()] == [(0, 0, 0), (0, 1, 0), (0, 1, 1)]
    v = orc.ray_voxels([0.5, 0.5, 0.5], [1.5, 1.5, 1.5], 1.0, 0.0)
    assert [tuple(r) for r in v.tolist()] == [(0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 1, 1)]


def test_floor_semantics_across_zero(orc):
    # floor, not truncation, across zero; start on a boundary moving negative
    v = orc.ray_voxels([-0.05, 0.05, 0.05], [-0.35, 0.05, 0.05], 0.1, 0.0)
    assert v[:, 0].tolist() == [-1, -2, -3, -4]
    v = orc.ray_voxels([1.0, 0.5, 0.5], [0.5, 0.5, 0.5], 1.0, 0.0)
    assert [tuple(r) for r in v.tolist()] == [(1, 0, 0), (0, 0, 0)]


def test_domain_limit(orc):
    # O3: |voxel| < 2^23 (21-bit block keys); beyond it the ray is rejected
    assert orc.ray_voxels([0, 0, 0], [0.1 * (1 << 23) + 1, 0, 0], 0.1, 0.0) is None
