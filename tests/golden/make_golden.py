"""Generate golden vectors by running the REAL reference package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small .npz fixtures next to this script.  `/root/reference` does not exist on
the GPU box; the fixtures travel instead.  Every case mirrors a reference test or a
SURVEY.md 8d configuration (citations inline).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from nfsense import Grid, grid_coordinates  # noqa: E402
from nfsense import engine, simulate, sensmaps, kfilter  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


def run_full(inputs, **kw):
    img, log = engine.recon_full(inputs, **kw)
    return img, log


def case_engine8():
    """tests/test_engine.py:30-36 small_setup + :154-165 split-vs-full (rng 1234)."""
    rng = np.random.default_rng(1234)
    grid = Grid((8, 8, 1), (0.08, 0.08, 0.002))
    n_coils, n_samples = 3, 90
    sens = rng.standard_normal((grid.nvox, n_coils)) + 1j * rng.standard_normal((grid.nvox, n_coils))
    temporal = simulate.make_spiral(n_samples, turns=4, k_max=320.0)
    coords = grid_coordinates(grid)
    spatial = np.vstack([simulate.make_b0(grid, "linear", 150.0), coords[:, :2].T])
    rho = rng.standard_normal(grid.nvox) + 1j * rng.standard_normal(grid.nvox)
    sig_rand = rng.standard_normal((n_samples, n_coils)) + 1j * rng.standard_normal((n_samples, n_coils))
    sigma = simulate.forward_signal(rng.standard_normal(grid.nvox) + 0j, sens, spatial, temporal,
                                    noise_sd=0.01, rng=rng)
    phase = engine.phase_block(temporal, spatial)
    mk = lambda starts=None, n_iter=15: engine.EncodingInputs(  # noqa: E731
        sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
        intensity=np.ones(grid.nvox), kfilter=None, mask_r=np.ones(grid.nvox, bool),
        grid=grid, n_iter=n_iter, block_starts=starts)
    full, flog = engine.recon_full(mk())
    starts = np.array([0, 13, 40, 41, 90])
    split, slog = engine.recon_split(mk(starts))
    save("engine8", sens=sens, temporal=temporal, spatial=spatial, rho=rho, sig_rand=sig_rand,
         sigma=sigma, phase_rows=engine.phase_block(temporal[10:20], spatial),
         E_rho=engine.apply_E(rho, sens, phase), EH_sig=engine.apply_EH(sig_rand, sens, phase),
         dense=simulate.dense_encoding_matrix(sens, spatial, temporal),
         full_values=full.values, full_res=np.array(flog.residual_norms),
         full_sol=np.array(flog.solution_norms), starts=starts, split_values=split.values,
         split_res=np.array(slog.residual_norms), split_sol=np.array(slog.solution_norms))


def case_oracle_eq():
    """tests/test_acceptance.py:74-103 (seed 2024); first 4 random instances."""
    rng = np.random.default_rng(2024)
    out = {}
    for i in range(4):
        n_vox = int(rng.integers(16, 257))
        n_samp = int(rng.integers(16, 513))
        n_coil = int(rng.integers(1, 5))
        n_terms = int(rng.integers(2, 16))
        spatial = rng.standard_normal((n_terms, n_vox))
        temporal = rng.standard_normal((n_samp, n_terms))
        sens = rng.standard_normal((n_vox, n_coil)) + 1j * rng.standard_normal((n_vox, n_coil))
        p = rng.standard_normal(n_vox) + 1j * rng.standard_normal(n_vox)
        sigma = rng.standard_normal((n_samp, n_coil)) + 1j * rng.standard_normal((n_samp, n_coil))
        phase = engine.phase_block(temporal, spatial)
        for key, val in dict(spatial=spatial, temporal=temporal, sens=sens, p=p, sigma=sigma,
                             E=engine.apply_E(p, sens, phase),
                             EH=engine.apply_EH(sigma, sens, phase)).items():
            out[f"{key}_{i}"] = val
    save("oracle_eq", **out)


def config_a_tables(mask):
    """SURVEY 8d config A via the reference's own generators (nfs/pipeline.py:21-117)."""
    grid = Grid((64, 64, 1), (0.22, 0.22, 0.002))
    traj = simulate.make_spiral(16384, turns=32, k_max=np.pi * 64 / 0.22, readout_s=0.03)
    b0 = simulate.make_b0(grid, "linear", 200.0)
    spatial, temporal = engine.build_bases(b0, mask, grid, traj[:, 0], traj[:, 1:], order=1)
    sens_full = simulate.synth_coils(grid, 8)
    return grid, traj, spatial, temporal, sens_full


def case_config_a():
    """Config A, 20 CG iterations, unmasked, and masked with j + k-space filter."""
    grid = Grid((64, 64, 1), (0.22, 0.22, 0.002))
    rho, support = simulate.make_phantom(grid, "discs", smooth_phase=True)
    ones = np.ones(grid.nvox, bool)
    grid, traj, spatial, temporal, sens_full = config_a_tables(ones)
    sigma = simulate.forward_signal(rho, sens_full, spatial, temporal)
    inputs = engine.EncodingInputs(sigma=sigma, spatial=spatial, temporal=temporal,
                                   sens=sens_full, intensity=np.ones(grid.nvox), kfilter=None,
                                   mask_r=ones, grid=grid, n_iter=20)
    img, log = engine.recon_full(inputs)
    rho_log = []
    inputs10 = engine.EncodingInputs(sigma=sigma, spatial=spatial, temporal=temporal,
                                     sens=sens_full, intensity=np.ones(grid.nvox), kfilter=None,
                                     mask_r=ones, grid=grid, n_iter=20)
    engine.recon_full(inputs10, callback=lambda n, r: rho_log.append(r.copy()))
    # masked variant: phantom support, intensity correction, convex-hull k filter
    _, _, spatial_m, temporal_m, _ = config_a_tables(support)
    j = sensmaps.intensity_correction(sens_full, support)[support]
    filt = kfilter.build_filter(traj[:, 1:3], grid)
    inputs_m = engine.EncodingInputs(sigma=sigma, spatial=spatial_m, temporal=temporal_m,
                                     sens=sens_full[support], intensity=j, kfilter=filt,
                                     mask_r=support, grid=grid, n_iter=20)
    rho_m_log = []
    img_m, log_m = engine.recon_full(inputs_m, callback=lambda n, r: rho_m_log.append(r.copy()))
    iters = np.array([5, 10, 15, 20])
    save("config_a", sigma=sigma, rho_true=rho, support=support,
         spatial_digest=np.array(digest(spatial)), temporal_digest=np.array(digest(temporal)),
         sens_digest=np.array(digest(sens_full)), spatial_rows=spatial[:, ::97],
         temporal_rows=temporal[::1021], sens_rows=sens_full[::131],
         values=img.values, res=np.array(log.residual_norms), sol=np.array(log.solution_norms),
         rho_iters=np.stack([rho_log[i - 1] for i in iters]), iters=iters,
         kfilter=filt, intensity=j, values_mask=img_m.values, res_mask=np.array(log_m.residual_norms),
         sol_mask=np.array(log_m.solution_norms),
         rho_iters_mask=np.stack([rho_m_log[i - 1] for i in iters]))


def case_small3d():
    """3D stack-of-spirals, order-3 harmonics (P+1=16), 4 coils, split and full."""
    grid = Grid((12, 12, 6), (0.22, 0.22, 0.128))
    rho, support = simulate.make_phantom(grid, "discs", smooth_phase=True)
    traj = simulate.make_spiral(150, turns=4, k_max=np.pi * 12 / 0.22, readout_s=0.03,
                                ndim=3, n_planes=6, kz_max=np.pi * 6 / 0.128)
    harm = simulate.solid_harmonics(3, grid_coordinates(grid), ndim=3)
    t = traj[:, 0]
    k_nyq = np.pi * min(n / f for n, f in zip(grid.dims, grid.fov_m))
    half = min(grid.fov_m) / 2
    extra = np.column_stack([0.05 * k_nyq / half ** (1 if p < 5 else 2)
                             * np.sin(2 * np.pi * (p + 1) * t / t[-1]) for p in range(12)])
    b0 = simulate.make_b0(grid, "linear", 200.0)
    spatial = np.vstack([b0[None], harm.T])
    temporal = np.column_stack([traj, extra])
    sens = simulate.synth_coils(grid, 4)
    sigma = simulate.forward_signal(rho, sens, spatial, temporal)
    mk = lambda starts=None: engine.EncodingInputs(  # noqa: E731
        sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
        intensity=np.ones(grid.nvox), kfilter=None, mask_r=np.ones(grid.nvox, bool),
        grid=grid, n_iter=12, block_starts=starts)
    full, flog = engine.recon_full(mk())
    starts = np.linspace(0, temporal.shape[0], 8, dtype=int)
    split, slog = engine.recon_split(mk(starts))
    save("small3d", spatial=spatial, temporal=temporal, sens=sens, sigma=sigma, rho_true=rho,
         values=full.values, res=np.array(flog.residual_norms), sol=np.array(flog.solution_norms),
         starts=starts, split_values=split.values, split_res=np.array(slog.residual_norms))


def case_cartesian8():
    """tests/test_engine.py:90-100 exact recovery with early stop."""
    grid = Grid((8, 8, 1), (0.08, 0.08, 0.002))
    rho, _ = simulate.make_phantom(grid, "discs", smooth_phase=True)
    sens = np.ones((grid.nvox, 1), complex)
    temporal = simulate.make_cartesian(grid)
    spatial = np.vstack([np.zeros(grid.nvox), grid_coordinates(grid)[:, :2].T])
    sigma = simulate.forward_signal(rho, sens, spatial, temporal)
    img, log = engine.recon_full(engine.EncodingInputs(
        sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
        intensity=np.ones(grid.nvox), kfilter=None, mask_r=np.ones(grid.nvox, bool),
        grid=grid, n_iter=10))
    save("cartesian8", temporal=temporal, sigma=sigma, rho_true=rho, values=img.values,
         res=np.array(log.residual_norms), iterations=np.array(img.iterations))


def case_config_b_rows():
    """Config B tables (256^2, 32 coils, P+1=16) and the operator on a row subset."""
    grid = Grid((256, 256, 1), (0.22, 0.22, 0.002))
    traj = simulate.make_spiral(65536, turns=32, k_max=np.pi * 256 / 0.22, readout_s=0.0715)
    c = grid_coordinates(grid)
    mask = np.hypot(c[:, 0], c[:, 1]) <= 0.45 * 0.22
    harm = simulate.solid_harmonics(3, c[mask], ndim=2)
    k_nyq = np.pi * 256 / 0.22
    t = traj[:, 0]
    extra = np.column_stack([0.05 * k_nyq / 0.11 ** (1 if p < 5 else 2)
                             * np.sin(2 * np.pi * (p + 1) * t / t[-1]) for p in range(13)])
    b0 = simulate.make_b0(grid, "linear", 200.0)
    spatial = np.vstack([b0[mask][None], harm.T])
    temporal = np.column_stack([traj, extra])
    sens_full = simulate.synth_coils(grid, 32)
    j = sensmaps.intensity_correction(sens_full, mask)[mask]
    sens = sens_full[mask] * j[:, None]
    rho, _ = simulate.make_phantom(grid, "discs", smooth_phase=True)
    rows = np.arange(0, 65536, 1024) + 7
    phase = engine.phase_block(temporal[rows], spatial)
    rng = np.random.default_rng(5)
    sig = rng.standard_normal((rows.size, 32)) + 1j * rng.standard_normal((rows.size, 32))
    save("config_b_rows", rows=rows, mask=mask, n_vox=np.array(mask.sum()),
         spatial_digest=np.array(digest(spatial)), temporal_digest=np.array(digest(temporal)),
         sens_digest=np.array(digest(sens)), spatial_cols=spatial[:, ::509],
         temporal_rows=temporal[rows], sens_rows=sens[::509], intensity_rows=j[::509],
         E_rows=engine.apply_E(rho[mask] / j, sens, phase), sig=sig,
         EH_rows=engine.apply_EH(sig, sens, phase).astype(np.complex128))


def config_b_problem():
    """Config B from the reference generators: tables, S, j, phantom."""
    grid = Grid((256, 256, 1), (0.22, 0.22, 0.002))
    traj = simulate.make_spiral(65536, turns=32, k_max=np.pi * 256 / 0.22, readout_s=0.0715)
    c = grid_coordinates(grid)
    mask = np.hypot(c[:, 0], c[:, 1]) <= 0.45 * 0.22
    harm = simulate.solid_harmonics(3, c[mask], ndim=2)
    k_nyq = np.pi * 256 / 0.22
    t = traj[:, 0]
    extra = np.column_stack([0.05 * k_nyq / 0.11 ** (1 if p < 5 else 2)
                             * np.sin(2 * np.pi * (p + 1) * t / t[-1]) for p in range(13)])
    b0 = simulate.make_b0(grid, "linear", 200.0)
    spatial = np.vstack([b0[mask][None], harm.T])
    temporal = np.column_stack([traj, extra])
    sens_full = simulate.synth_coils(grid, 32)
    j = sensmaps.intensity_correction(sens_full, mask)[mask]
    rho, _ = simulate.make_phantom(grid, "discs", smooth_phase=True)
    return grid, mask, spatial, temporal, sens_full[mask], j, rho[mask]


def blocked_forward(rho, sens, spatial, temporal, budget=2 ** 28):
    """sigma = E rho through the reference's own phase_block / apply_E, block by block."""
    starts = engine.choose_block_starts(temporal.shape[0], spatial.shape[1], budget)
    out = [engine.apply_E(rho, sens, engine.phase_block(temporal[lo:hi], spatial))
           for lo, hi in zip(starts[:-1], starts[1:])]
    return np.concatenate(out, axis=0)


def case_config_b_cg():
    """Config B CG through the reference recon_split (nfs/engine.py:182-241) with the
    pipeline's 2^28-byte blocks (nfs/pipeline.py:221), 10 iterations, noiseless phantom
    data (sigma = E rho_true with the unnormalised coil maps).  ~40 min of CPU."""
    grid, mask, spatial, temporal, sens, j, rho = config_b_problem()
    sigma = blocked_forward(rho, sens, spatial, temporal)
    starts = engine.choose_block_starts(temporal.shape[0], spatial.shape[1], 2 ** 28)
    inputs = engine.EncodingInputs(sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
                                   intensity=j, kfilter=None, mask_r=mask, grid=grid,
                                   n_iter=10, block_starts=starts)
    rho_log = {}
    img, log = engine.recon_split(inputs, callback=lambda n, r: rho_log.__setitem__(n, r.copy()))
    iters = np.array([1, 5, 10])
    rows = np.arange(0, 65536, 2048) + 5
    save("config_b_cg", mask=mask, spatial_digest=np.array(digest(spatial)),
         temporal_digest=np.array(digest(temporal)), sens_digest=np.array(digest(sens)),
         j_rows=j[::509], rho_true=rho, sigma_rows=sigma[rows], rows=rows, starts=starts,
         iters=iters, rho_iters=np.stack([rho_log[i] for i in iters]), values=img.values,
         res=np.array(log.residual_norms), sol=np.array(log.solution_norms))


def config_d_problem(scale=4):
    """Config D scaled down in every axis by `scale`: 3D stack of spirals,
    order-3 solid harmonics (P+1 = 16), 32 coils, ellipsoid mask (~50 %), built from the
    reference generators the way nfs/pipeline.py:21-117 assembles a 3D problem."""
    nxy, nz = 128 // scale, 64 // scale
    grid = Grid((nxy, nxy, nz), (0.22, 0.22, 0.128))
    traj = simulate.make_spiral(4682 // scale ** 2, turns=9.14 / scale, k_max=np.pi * nxy / 0.22,
                                readout_s=0.03, ndim=3, n_planes=nz, kz_max=np.pi * nz / 0.128)
    c = grid_coordinates(grid)
    mask = (c[:, 0] / 0.11) ** 2 + (c[:, 1] / 0.11) ** 2 + (c[:, 2] / 0.064) ** 2 <= 0.98
    harm = simulate.solid_harmonics(3, c[mask], ndim=3)
    k_nyq = np.pi * min(n / f for n, f in zip(grid.dims, grid.fov_m))
    half = min(grid.fov_m) / 2
    t = traj[:, 0]
    extra = np.column_stack([0.05 * k_nyq / half ** (1 if p < 5 else 2)
                             * np.sin(2 * np.pi * (p + 1) * t / t[-1]) for p in range(12)])
    b0 = simulate.make_b0(grid, "linear", 200.0)
    spatial = np.vstack([b0[mask][None], harm.T])
    temporal = np.column_stack([traj, extra])
    sens_full = simulate.synth_coils(grid, 32)
    j = sensmaps.intensity_correction(sens_full, mask)[mask]
    rho, _ = simulate.make_phantom(grid, "discs", smooth_phase=True)
    return grid, mask, spatial, temporal, sens_full[mask], j, rho[mask]


def case_config_d_small():
    """Config D at 32x32x16 (scale 4): 32 coils, P+1 = 16, 50 CG iterations through the
    reference recon_full (nfs/engine.py:125-179) -- SURVEY 8d's full-iteration 3D parity."""
    grid, mask, spatial, temporal, sens, j, rho = config_d_problem(4)
    sigma = blocked_forward(rho, sens, spatial, temporal)
    inputs = engine.EncodingInputs(sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
                                   intensity=j, kfilter=None, mask_r=mask, grid=grid, n_iter=50)
    rho_log = {}
    img, log = engine.recon_full(inputs, callback=lambda n, r: rho_log.__setitem__(n, r.copy()))
    iters = np.array([1, 5, 10, 20, 30, 50])
    save("config_d_small", mask=mask, spatial_digest=np.array(digest(spatial)),
         temporal_digest=np.array(digest(temporal)), sens_digest=np.array(digest(sens)),
         j=j, rho_true=rho, sigma=sigma.astype(np.complex64), sigma_digest=np.array(digest(sigma)),
         iters=iters, rho_iters=np.stack([rho_log[i] for i in iters]), values=img.values,
         res=np.array(log.residual_norms), sol=np.array(log.solution_norms))


def case_config_c_slice():
    """Config C: one off-centre slice (z = +39 mm, slice 39 of a 40-slice stack at
    2 mm spacing) of config B scaled to 64x64 (scale 4): the third-order harmonics at z != 0,
    shared trajectory, 32 coils, slice contrast 1.25; reference recon_full, 10 iterations."""
    scale, z = 4, 0.002 * (39 - 19.5)
    n = 256 // scale
    grid = Grid((n, n, 1), (0.22, 0.22, 0.002))
    traj = simulate.make_spiral(65536 // scale ** 2, turns=32 / scale, k_max=np.pi * n / 0.22,
                                readout_s=0.0715)
    c = grid_coordinates(grid)
    mask = np.hypot(c[:, 0], c[:, 1]) <= 0.45 * 0.22
    cz = c[mask].copy()
    cz[:, 2] += z
    harm = simulate.solid_harmonics(3, cz, ndim=2)
    k_nyq = np.pi * n / 0.22
    t = traj[:, 0]
    extra = np.column_stack([0.05 * k_nyq / 0.11 ** (1 if p < 5 else 2)
                             * np.sin(2 * np.pi * (p + 1) * t / t[-1]) for p in range(13)])
    b0 = simulate.make_b0(grid, "linear", 200.0)
    spatial = np.vstack([b0[mask][None], harm.T])
    temporal = np.column_stack([traj, extra])
    sens_full = simulate.synth_coils(grid, 32)
    j = sensmaps.intensity_correction(sens_full, mask)[mask]
    rho, _ = simulate.make_phantom(grid, "discs", smooth_phase=True)
    rho = rho[mask] * 1.25
    sens = sens_full[mask]
    sigma = blocked_forward(rho, sens, spatial, temporal)
    inputs = engine.EncodingInputs(sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
                                   intensity=j, kfilter=None, mask_r=mask, grid=grid, n_iter=10)
    rho_log = {}
    img, log = engine.recon_full(inputs, callback=lambda n, r: rho_log.__setitem__(n, r.copy()))
    iters = np.array([1, 5, 10])
    save("config_c_slice", mask=mask, spatial_digest=np.array(digest(spatial)),
         temporal_digest=np.array(digest(temporal)), sens_digest=np.array(digest(sens)), z=np.array(z),
         rho_true=rho, sigma=sigma.astype(np.complex64), iters=iters,
         rho_iters=np.stack([rho_log[i] for i in iters]), values=img.values,
         res=np.array(log.residual_norms), sol=np.array(log.solution_norms))


def case_config_d_small_split():
    """The reference's OWN sensitivity on the config-D-small CG: recon_split (4 row blocks) vs
    recon_full differ only by summation order, so their iterate drift over 50 iterations is the
    floor any other FP64 implementation can be held to."""
    grid, mask, spatial, temporal, sens, j, rho = config_d_problem(4)
    sigma = blocked_forward(rho, sens, spatial, temporal)
    starts = np.linspace(0, temporal.shape[0], 5, dtype=int)
    inputs = engine.EncodingInputs(sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
                                   intensity=j, kfilter=None, mask_r=mask, grid=grid, n_iter=50,
                                   block_starts=starts)
    rho_log = {}
    img, log = engine.recon_split(inputs, callback=lambda n, r: rho_log.__setitem__(n, r.copy()))
    iters = np.array([1, 5, 10, 20, 30, 50])
    save("config_d_small_split", starts=starts, iters=iters,
         rho_iters=np.stack([rho_log[i] for i in iters]), res=np.array(log.residual_norms))


def case_metrics():
    """nfs/metrics.py ssim / rmse (tests/test_metrics.py) on the images a convergence study
    compares: a 24x20 magnitude image vs a reference, with and without a window mask."""
    from nfsense import metrics
    rng = np.random.default_rng(13)
    ref = np.abs(rng.standard_normal((24, 20))) + np.linspace(0, 2, 20)[None, :]
    test = ref + 0.2 * rng.standard_normal((24, 20))
    mask = rng.random((24, 20)) < 0.6
    m_plain, smap_plain = metrics.ssim(test, ref)
    m_mask, _ = metrics.ssim(test, ref, mask=mask)
    m_w5, smap_w5 = metrics.ssim(test, ref, window=5, sigma=1.5)
    full_ref = rng.standard_normal(300) + 1j * rng.standard_normal(300)
    full_test = full_ref + 0.1 * (rng.standard_normal(300) + 1j * rng.standard_normal(300))
    sup = rng.random(300) < 0.5
    save("metrics", ref=ref, test=test, mask=mask, ssim_plain=np.array(m_plain), smap_plain=smap_plain,
         ssim_mask=np.array(m_mask), ssim_w5=np.array(m_w5), smap_w5=smap_w5, full_ref=full_ref,
         full_test=full_test, support=sup, rmse=np.array(metrics.rmse(full_test, full_ref, sup)))


if __name__ == "__main__":
    which = sys.argv[1:] or ["engine8", "oracle_eq", "config_a", "small3d", "cartesian8",
                             "config_b_rows", "metrics"]
    for name in which:
        globals()["case_" + name]()
