"""Pins of the oracle's ESDF and query (O13).

References: a literal brute-force minimum over sites, scipy.ndimage.distance_transform_edt (a library
exact EDT), single-site and plane-of-sites closed forms, the voxel-centre identity of trilinear
interpolation and exactness of trilinear interpolation on affine fields.
"""
import numpy as np
import pytest
from scipy import ndimage


def _random_tsdf(rng, nb_side=(3, 3, 2), fill=0.8, p_obs=0.9, tau=0.3):
    blocks = [(x, y, z) for x in range(nb_side[0]) for y in range(nb_side[1]) for z in range(nb_side[2])
              if rng.random() < fill]
    b = np.array(blocks, np.int32) - np.array([1, 1, 0], np.int32)
    nb = len(blocks)
    W = (rng.random((nb, 512)) < p_obs).astype(np.float64) * rng.uniform(0.5, 3, (nb, 512))
    D = rng.uniform(-tau, tau, (nb, 512)) * (W > 0)
    return b, D, W


def _dense(b, vals, fill):
    lo = b.min(0) * 8
    hi = b.max(0) * 8 + 8
    G = np.full(tuple(hi - lo), fill, dtype=vals.dtype)
    l = np.arange(512)
    for i in range(b.shape[0]):
        G[8 * b[i, 0] - lo[0] + l % 8, 8 * b[i, 1] - lo[1] + (l // 8) % 8, 8 * b[i, 2] - lo[2] + l // 64] = vals[i]
    return G, lo


@pytest.mark.parametrize("seed", range(3))
def test_separable_equals_brute_force_and_scipy(orc, seed):
    rng = np.random.default_rng(seed)
    b, D, W = _random_tsdf(rng)
    s, thr = 0.1, 0.02
    E_sep, d2_sep = orc.esdf(b, D, W, s, thr, brute=False)
    E_bf, d2_bf = orc.esdf(b, D, W, s, thr, brute=True)
    assert np.array_equal(d2_sep, d2_bf)
    # scipy: distance to the nearest zero of ~site over the dense AABB (unallocated -> not a site)
    site = (W > 0) & (np.abs(D) <= thr)
    G, lo = _dense(b, site, False)
    ref = ndimage.distance_transform_edt(~G)
    l = np.arange(512)
    for i in range(b.shape[0]):
        r = ref[8 * b[i, 0] - lo[0] + l % 8, 8 * b[i, 1] - lo[1] + (l // 8) % 8, 8 * b[i, 2] - lo[2] + l // 64]
        assert np.array_equal(np.rint(r * r).astype(np.int64), d2_sep[i])
    obs = W > 0
    assert np.isnan(E_sep[~obs]).all()
    assert np.allclose(np.abs(E_sep[obs]), s * np.sqrt(d2_sep[obs]), rtol=0, atol=1e-12)
    assert (np.sign(E_sep[obs & (D < 0) & (d2_sep > 0)]) < 0).all()
    assert (E_sep[obs & (D >= 0)] >= 0).all()


def test_single_site_and_plane(orc):
    s = 0.05
    b = np.array([[x, y, z] for x in range(-1, 2) for y in range(-1, 2) for z in range(0, 2)], np.int32)
    nb = len(b)
    W = np.ones((nb, 512))
    D = np.full((nb, 512), 0.2)
    # single site at voxel (3, -5, 9)
    l = np.arange(512)
    vx = 8 * b[:, 0:1] + l % 8
    vy = 8 * b[:, 1:2] + (l // 8) % 8
    vz = 8 * b[:, 2:3] + l // 64
    Ds = D.copy()
    Ds[(vx == 3) & (vy == -5) & (vz == 9)] = 0.0
    E, d2 = orc.esdf(b, Ds, W, s, 0.01)
    assert np.allclose(E, s * np.sqrt((vx - 3) ** 2 + (vy + 5) ** 2 + (vz - 9) ** 2), atol=1e-12)
    # plane of sites at layer z = 6, negative below
    Dp = np.where(vz == 6, 0.0, np.where(vz < 6, -0.2, 0.2))
    E, d2 = orc.esdf(b, Dp, W, s, 0.01)
    assert np.allclose(E, np.sign(vz - 6) * s * np.abs(vz - 6), atol=1e-12)


def test_empty_site_set_and_unobserved(orc):
    b = np.array([[0, 0, 0], [1, 0, 0]], np.int32)
    W = np.ones((2, 512))
    W[1, :10] = 0
    D = np.full((2, 512), 0.3)
    E, d2 = orc.esdf(b, D, W, 0.1, 0.1)
    assert np.isposinf(E[W > 0]).all() and np.isnan(E[W == 0]).all()
    assert (d2 == -1).all()


def _affine_blocks(a, s):
    b = np.array([[x, y, z] for x in range(-1, 2) for y in range(-1, 2) for z in range(-1, 2)], np.int32)
    l = np.arange(512)
    vx = 8 * b[:, 0:1] + l % 8
    vy = 8 * b[:, 1:2] + (l // 8) % 8
    vz = 8 * b[:, 2:3] + l // 64
    c = np.stack([(vx + 0.5) * s, (vy + 0.5) * s, (vz + 0.5) * s], -1)
    E = c @ a[:3] + a[3]
    return b, E


def test_query_voxel_centre_identity_and_affine_exactness(orc):
    s = 0.25                                  # dyadic: voxel centres are exact, f = 0 exactly
    a = np.array([0.3, -1.1, 0.7, 0.05])
    b, E = _affine_blocks(a, s)
    rng = np.random.default_rng(0)
    # at a voxel centre the interpolation returns the stored value exactly
    v = rng.integers(-7, 7, (200, 3))
    pts = ((v + 0.5) * s).astype(np.float32)
    val, st = orc.query(b, E, s, np.eye(4), pts)
    assert (st == 0).all()
    l = (v % 8)[:, 0] + 8 * (v % 8)[:, 1] + 64 * (v % 8)[:, 2]
    blk = {tuple(k): i for i, k in enumerate(b.tolist())}
    ref = np.array([E[blk[tuple((vv // 8).tolist())], ll] for vv, ll in zip(v, l)])
    assert np.array_equal(val, ref)
    # trilinear interpolation is exact on an affine field
    x = rng.uniform(-7 * s, 7 * s, (500, 3)).astype(np.float32)
    val, st = orc.query(b, E, s, np.eye(4), x)
    assert (st == 0).all()
    assert np.allclose(val, x.astype(np.float64) @ a[:3] + a[3], atol=1e-9)


def test_query_status_and_pose(orc):
    s = 0.25
    a = np.array([0.0, 0.0, 1.0, 0.0])
    b, E = _affine_blocks(a, s)
    E = E.copy()
    E[13, 0] = np.nan                        # one unobserved voxel in block (0,0,0) at local 0
    T = np.eye(4)
    T[:3, 3] = [1.0, -2.0, 0.5]
    # a point whose 8-corner stencil includes the unobserved voxel (0,0,0) but whose own voxel is (0,0,0)
    # -> UNKNOWN;  a point whose own voxel is observed but whose stencil touches (0,0,0) -> NEAREST
    pts_s = np.array([[0.1, 0.1, 0.1], [0.3, 0.3, 0.3], [10.0, 10.0, 10.0], [0.6, 0.6, 0.6]])
    pts_w = (pts_s + T[:3, 3]).astype(np.float32)
    val, st = orc.query(b, E, s, T, pts_w)
    assert st.tolist() == [2, 1, 2, 0]
    assert np.isnan(val[0]) and np.isnan(val[2])
    assert val[1] == pytest.approx(E[13, 1 + 8 + 64])


def test_esdf_sample_equals_full_transform(orc):
    rng = np.random.default_rng(9)
    b, D, W = _random_tsdf(rng)
    E, d2 = orc.esdf(b, D, W, 0.1, 0.02, brute=True)
    l = np.arange(512)
    vox = np.stack([8 * b[:, 0:1] + l % 8, 8 * b[:, 1:2] + (l // 8) % 8, 8 * b[:, 2:3] + l // 64], -1).reshape(-1, 3)
    pick = rng.choice(vox.shape[0], 300, replace=False)
    s = orc.esdf_sample(b, D, W, 0.02, vox[pick])
    assert np.array_equal(s, d2.reshape(-1)[pick])


def test_query_gradient_affine_and_finite_differences(orc):
    """f4 pin: on an affine field the trilinear gradient is the field's gradient (rotated to world);
    elsewhere it matches central finite differences of the interpolated value inside a cell."""
    s = 0.25
    a = np.array([0.3, -1.1, 0.7, 0.05])
    b, E = _affine_blocks(a, s)
    import synth
    T = synth.pose(synth.rot_zyx(0.4, 0.1, -0.2), [0.5, -0.25, 0.1])
    rng = np.random.default_rng(3)
    xs = rng.uniform(-6 * s, 6 * s, (300, 3))
    xw = (xs @ T[:3, :3].T + T[:3, 3]).astype(np.float32)
    val, st, g = orc.query(b, E, s, T, xw, gradient=True)
    assert (st == 0).all()
    assert np.allclose(g, np.tile(T[:3, :3] @ a[:3], (300, 1)), atol=1e-9)
    # non-affine field: finite differences of the interpolant along random world directions
    rng2 = np.random.default_rng(4)
    E2 = rng2.normal(size=E.shape)
    x0 = rng.uniform(-5 * s, 5 * s, (50, 3))
    h = 1e-4
    for d in np.eye(3):
        xp = ((x0 + h * d) @ T[:3, :3].T + T[:3, 3])
        xm = ((x0 - h * d) @ T[:3, :3].T + T[:3, 3])
        x_ = (x0 @ T[:3, :3].T + T[:3, 3])
        vp, _ = orc.query(b, E2, s, T, xp)
        vm, _ = orc.query(b, E2, s, T, xm)
        _, _, g2 = orc.query(b, E2, s, T, x_, gradient=True)
        fd = (vp - vm) / (2 * h)                                     # derivative along submap axis d
        assert np.allclose(g2 @ T[:3, :3] @ d, fd, atol=2e-2)


def test_sample_surface_proportional_and_brute_force(orc):
    """f4 pin: picks follow the weight distribution (exact counts for evenly spaced uniforms) and equal a
    brute-force linear search over the candidate list."""
    rng = np.random.default_rng(8)
    b, D, W = _random_tsdf(rng)
    W = np.round(W * 3)                                 # integer weights (constant-weight fusion)
    thr = 0.05
    site = (W > 0) & (np.abs(D) <= thr)
    m = 4096
    u = (np.arange(m, dtype=np.uint64) * (1 << 32) // m).astype(np.uint32)
    xyz, w, tot = orc.sample_surface(b, D, W, thr, 0.1, np.eye(4), u)
    assert tot == int((W[site] * (1 << 20)).sum())
    # brute force: candidates in lexicographic block order, then local order
    order = np.lexsort((b[:, 2], b[:, 1], b[:, 0]))
    cand, wts = [], []
    l = np.arange(512)
    for ob in order:
        for li in l[site[ob]]:
            cand.append(((8 * b[ob, 0] + li % 8 + 0.5) * 0.1, (8 * b[ob, 1] + (li // 8) % 8 + 0.5) * 0.1,
                         (8 * b[ob, 2] + li // 64 + 0.5) * 0.1))
            wts.append(int(W[ob, li]) << 20)
    cum = np.cumsum(wts)
    tgt = (tot * u.astype(object)) // (1 << 32)
    ks = [int(np.searchsorted(cum, int(t), side="right")) for t in tgt]
    assert np.allclose(xyz, np.array(cand, np.float32)[ks], atol=1e-6)
    # proportionality: evenly spaced uniforms hit each candidate about w_k / T * m times
    counts = np.bincount(ks, minlength=len(cand))
    assert np.abs(counts - np.array(wts) / tot * m).max() <= 1.0 + 1e-9


@pytest.mark.parametrize("seed", range(3))
def test_capped_esdf_pins(orc, seed):
    """f1's value (R11): O11 clamped at d_max.  Pinned against scipy's exact EDT on the dense AABB
    (independent of orc_esdf), single-site closed form, empty site set -> +-d_max, brute == separable, and
    an infinite cap reproducing the uncapped O11 exactly."""
    rng = np.random.default_rng(100 + seed)
    b, D, W = _random_tsdf(rng, nb_side=(4, 3, 2), fill=0.7)
    s, thr, dmax = 0.1, 0.01, 0.45
    Ec = orc.esdf_capped(b, D, W, s, thr, dmax)
    assert np.array_equal(Ec, orc.esdf_capped(b, D, W, s, thr, dmax, brute=True), equal_nan=True)
    site = (W > 0) & (np.abs(D) <= thr)
    G, lo = _dense(b, site, False)
    ref = ndimage.distance_transform_edt(~G) * s
    l = np.arange(512)
    obs = W > 0
    for i in range(b.shape[0]):
        r = ref[8 * b[i, 0] - lo[0] + l % 8, 8 * b[i, 1] - lo[1] + (l // 8) % 8, 8 * b[i, 2] - lo[2] + l // 64]
        want = np.where(D[i] < 0, -1.0, 1.0) * np.minimum(r, dmax)
        o = obs[i]
        assert np.allclose(Ec[i][o], want[o], rtol=0, atol=1e-12)
        assert np.isnan(Ec[i][~o]).all()
    assert np.nanmax(np.abs(Ec)) == dmax                      # the cap binds somewhere in this scene
    E, _ = orc.esdf(b, D, W, s, thr)
    assert np.array_equal(orc.esdf_capped(b, D, W, s, thr, np.inf), E, equal_nan=True)
    # no site at all: every observed voxel holds +-d_max
    Dn = np.where(W > 0, np.where(D < 0, -0.2, 0.2), 0.0)
    En = orc.esdf_capped(b, Dn, W, s, thr, dmax)
    assert np.array_equal(np.abs(En[obs]), np.full(obs.sum(), dmax))
    assert (np.signbit(En[obs]) == (Dn[obs] < 0)).all()
    # one site: closed form min(s |v - u|, d_max)
    D1 = np.full_like(D, 0.2)
    W1 = np.ones_like(W)
    D1[0, 3 + 8 * 2 + 64 * 5] = 0.0
    u = 8 * b[0] + np.array([3, 2, 5])
    E1 = orc.esdf_capped(b, D1, W1, s, thr, dmax)
    for i in range(b.shape[0]):
        v = 8 * b[i][None, :] + np.stack([l % 8, (l // 8) % 8, l // 64], 1)
        assert np.allclose(E1[i], np.minimum(s * np.linalg.norm(v - u, axis=1), dmax), rtol=0, atol=1e-12)
