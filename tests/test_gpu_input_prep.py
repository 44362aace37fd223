"""Input preparation on the device: intensity correction and mask restriction.

The reference computes j = 1/sqrt(sum_c |S|^2) on the host (nfs/sensmaps.py:145-152) and
restricts the maps to the reconstruction mask (nfs/pipeline.py:202-203); here both run on the GPU
(`engine.intensity_correction`, `engine.DeviceSens`).  j is checked against the reference's own
values in the golden fixtures (masked config A, config D scaled), and a reconstruction fed with
the full-grid maps must equal the one fed with host-restricted maps bit for bit.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

from paper_2604_09233_b200 import engine, simulate  # noqa: E402
from paper_2604_09233_b200.core import grid_coordinates  # noqa: E402


def _coils_full(grid, n):
    return simulate.synth_coils(grid, n)


def test_device_intensity_correction_matches_reference_config_a():
    g = golden("config_a")
    pm = simulate.make_problem("A_mask")
    j_full = engine.intensity_correction(_coils_full(pm.grid, 8), pm.mask_r)
    assert np.all(j_full[~pm.mask_r] == 0)
    assert np.allclose(j_full[pm.mask_r], g["intensity"], rtol=1e-15, atol=0)


def test_device_intensity_correction_matches_reference_config_d():
    g = golden("config_d_small")
    prob = simulate.make_problem("D", scale=4)
    h = engine.DeviceSens(_coils_full(prob.grid, 32), prob.mask_r)
    assert h.shape == prob.sens.shape
    assert np.array_equal(np.asarray(h), prob.sens)                  # host view = restriction
    assert np.allclose(h.intensity, g["j"], rtol=1e-15, atol=0)


@pytest.mark.parametrize("prec", ["fp64", "f16x3"])
def test_full_grid_maps_give_the_same_reconstruction(prec):
    g = golden("config_a")
    pm = simulate.make_problem("A_mask")
    full = _coils_full(pm.grid, 8)
    dev = engine.DeviceSens(full, pm.mask_r)
    mk = lambda sens, j: engine.EncodingInputs(  # noqa: E731
        sigma=g["sigma"], spatial=pm.spatial, temporal=pm.temporal, sens=sens, intensity=j, kfilter=None,
        mask_r=pm.mask_r, grid=pm.grid, n_iter=8)
    a, la = engine.recon_full(mk(pm.sens, pm.intensity), precision=prec)
    b, lb = engine.recon_full(mk(dev, pm.intensity), precision=prec)
    assert np.array_equal(a.values, b.values)
    assert la.residual_norms == lb.residual_norms
    # j from the device as well: equal to the reference's j to the last bits, so the images agree
    c, _ = engine.recon_full(mk(dev, dev.intensity), precision=prec)
    assert np.linalg.norm(c.values - a.values) <= 1e-13 * np.linalg.norm(a.values)


def test_voxel_index_outside_grid_rejected():
    pm = simulate.make_problem("A_mask")
    bad = engine.DeviceSens(_coils_full(pm.grid, 8), pm.mask_r)
    bad.vox_index = bad.vox_index.copy()
    bad.vox_index[0] = pm.grid.nvox + 5
    with pytest.raises(engine.EngineError):
        bad.intensity
    assert grid_coordinates(pm.grid).shape[0] == pm.grid.nvox
