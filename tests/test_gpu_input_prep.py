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


def _write_dataset(tmp_path, sigma):
    """A dataset directory in the reference's on-disk format (nfs/core.py:292-328): raw
    little-endian complex128 + manifest.json."""
    import json
    np.ascontiguousarray(sigma, dtype="<c16").tofile(tmp_path / "sigma.c128")
    (tmp_path / "manifest.json").write_text(json.dumps(
        {"version": 1, "grid": {"dims": [64, 64, 1], "fov_m": [0.22, 0.22, 0.002]}, "counts": {},
         "echo_times_s": [], "byte_order": "little", "element_order": "x-fastest",
         "arrays": {"sigma": {"file": "sigma.c128", "dtype": "c128", "shape": list(sigma.shape)}}}))
    return tmp_path


@pytest.mark.parametrize("prec", ["fp64", "f16x3"])
def test_samples_read_from_dataset_file(tmp_path, prec):
    """the raw samples go from the dataset file to the device through the pinned
    ring (nfs_set_samples_file) -- same reconstruction, bit for bit, as from a host array."""
    g = golden("config_a")
    pm = simulate.make_problem("A_mask")
    ds = engine.DatasetSamples(_write_dataset(tmp_path, g["sigma"]))
    assert ds.shape == g["sigma"].shape and np.array_equal(np.asarray(ds), g["sigma"])
    mk = lambda sig: engine.EncodingInputs(  # noqa: E731
        sigma=sig, spatial=pm.spatial, temporal=pm.temporal, sens=pm.sens, intensity=pm.intensity,
        kfilter=None, mask_r=pm.mask_r, grid=pm.grid, n_iter=8)
    a, la = engine.recon_full(mk(g["sigma"]), precision=prec)
    b, lb = engine.recon_full(mk(ds), precision=prec)
    assert np.array_equal(a.values, b.values) and la.residual_norms == lb.residual_norms


def test_sample_rows_of_a_shard_from_file(tmp_path):
    """A sharded rank reads only rows [lo, hi) of the file: the shard plan's adjoint equals the
    one fed with the same rows from memory."""
    from paper_2604_09233_b200._native import Plan
    g = golden("config_a")
    pm = simulate.make_problem("A_mask")
    path = _write_dataset(tmp_path, g["sigma"]) / "sigma.c128"
    k = pm.temporal.shape[0]
    lo, hi = engine.shard_rows(k, 1, 3)
    outs = []
    for from_file in (False, True):
        plan = Plan(hi - lo, pm.spatial.shape[1], 8, 3, "fp64")
        plan.set_tables(pm.temporal[lo:hi], pm.spatial)
        plan.set_sens(pm.sens, pm.intensity)
        if from_file:
            plan.set_samples_file(str(path), lo)
        else:
            plan.set_samples(g["sigma"][lo:hi])
        outs.append(plan.cg_solve(3)[0])
        plan.close()
    assert np.array_equal(outs[0], outs[1])
    bad = Plan(hi - lo, pm.spatial.shape[1], 8, 3, "fp64")
    bad.set_tables(pm.temporal[lo:hi], pm.spatial)
    bad.set_sens(pm.sens, pm.intensity)
    with pytest.raises(engine.EngineError):
        bad.set_samples_file(str(path), k - 10)          # runs past the end of the file
    bad.close()
