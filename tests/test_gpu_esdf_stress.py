"""ESDF stress (BASELINE.json configs[4]) at reduced extent: a fully observed 2 cm TSDF imported from an
analytic SDF, exact ESDF vs the oracle's separable EDT on the same (exported) TSDF, and re-finalize
(recompute) idempotence."""
import numpy as np
import pytest
import torch

from helpers import assert_esdf_parity, gpu_export_sorted

pytestmark = pytest.mark.gpu


def test_esdf_stress_small_parity(orc):
    import synth.scenes as S
    from paper_2410_21149_b200 import Submap
    dev = torch.device("cuda", 0)
    s, tau = 0.02, 0.06
    sm = Submap(dict(voxel_size=s, truncation=tau, site_threshold=s, max_blocks=1 << 17), np.eye(4), 0)
    nb = 0
    for b, D, W in S.esdf_stress_blocks(voxel_size=s, truncation=tau, extent=(6.0, 6.0, 1.6), device=dev,
                                         n_boxes=5, n_spheres=4):
        sm.import_tsdf(b, D, W)
        nb += b.shape[0]
    sm.finalize_esdf()
    bg, Dg, Wg, Eg = gpu_export_sorted(sm)
    assert bg.shape[0] == nb
    Eo, _ = orc.esdf(bg, Dg.astype(np.float64), Wg.astype(np.float64), s, s)
    assert_esdf_parity(Eg, Eo, Wg > 0)
    assert (Eg < 0).any() and (Eg > 0.1).any()
    sm.finalize_esdf()                                   # recompute: identical
    _, _, _, E2 = gpu_export_sorted(sm)
    assert np.array_equal(E2.view(np.uint32), Eg.view(np.uint32))
