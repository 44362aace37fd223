"""Synthetic inputs for the benchmark configurations.

Host-side table builders that feed the device path: trajectories (temporal basis),
solid-harmonic spatial basis, phantom, coil maps and B0 maps.  They follow the
reference's generators (`nfs/simulate.py:26-212`, `nfs/pipeline.py:21-117`) so that
the same inputs reach both the CUDA path and the CPU oracle; golden tests pin them
to the reference's own outputs.  The raw samples for large configurations are
synthesised on the GPU by the forward operator itself.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import Grid, grid_coordinates


def solid_harmonics(order: int, coords: np.ndarray, ndim: int = 3,
                    include_constant: bool = False) -> np.ndarray:
    """Zero-Laplacian polynomial terms (nfs/simulate.py:26-59): 2/3, 8, 15 columns."""
    if order not in (1, 2, 3):
        raise ValueError(f"unsupported order {order}")
    c = np.asarray(coords, dtype=float)
    x, y, z = c[:, 0], c[:, 1], c[:, 2]
    out = []
    if include_constant:
        out.append(np.ones_like(x))
    out.extend([x, y] if (ndim == 2 and order == 1) else [x, y, z])
    if order >= 2:
        out.extend([x * y, z * y, 2 * z**2 - x**2 - y**2, z * x, x**2 - y**2])
    if order >= 3:
        out.extend([
            y * (3 * x**2 - y**2), x * y * z, y * (4 * z**2 - x**2 - y**2),
            z * (2 * z**2 - 3 * x**2 - 3 * y**2), x * (4 * z**2 - x**2 - y**2),
            z * (x**2 - y**2), x * (x**2 - 3 * y**2),
        ])
    return np.column_stack(out)


def make_spiral(n_samples, turns, k_max, readout_s=0.03, ndim=2, n_planes=1, kz_max=0.0):
    """Archimedean spiral-out temporal basis [t, kx, ky(, kz)] (nfs/simulate.py:165-187)."""
    if n_samples < 2:
        raise ValueError("need at least 2 samples")
    t = np.linspace(0.0, readout_s, n_samples)
    frac = t / readout_s
    ang = 2 * np.pi * turns * frac
    kx, ky = k_max * frac * np.cos(ang), k_max * frac * np.sin(ang)
    if ndim == 2:
        return np.column_stack([t, kx, ky])
    kzs = np.linspace(-kz_max, kz_max, n_planes) if n_planes > 1 else np.array([0.0])
    return np.vstack([np.column_stack([t, kx, ky, np.full(n_samples, kz)]) for kz in kzs])


def make_cartesian(grid: Grid, undersample=1, axis=1, readout_s=0.03):
    """Centred FFT-grid raster keeping every R-th line (nfs/simulate.py:190-212)."""
    nd = grid.ndim
    ks = [(2 * np.pi / fov) * (np.arange(n) - n // 2)
          for n, fov in zip(grid.dims[:nd], grid.fov_m[:nd])]
    ks[axis] = ks[axis][::undersample]
    mesh = np.meshgrid(*ks, indexing="ij")
    pts = np.column_stack([m.ravel(order="F") for m in mesh])
    return np.column_stack([np.linspace(0.0, readout_s, pts.shape[0]), pts])


def make_phantom(grid: Grid, kind="discs", smooth_phase=False):
    """Disc phantom with known support (nfs/simulate.py:66-120, kind 'discs')."""
    if kind != "discs":
        raise ValueError("only the 'discs' phantom is used by the benchmark configs")
    c = grid_coordinates(grid)
    x, y = c[:, 0], c[:, 1]
    rx, ry = grid.fov_m[0] / 2, grid.fov_m[1] / 2
    img = np.zeros(grid.nvox)
    for cx, cy, rad, val in ((0.0, 0.0, 0.72, 1.0), (-0.3, -0.25, 0.28, 0.6),
                             (0.32, 0.18, 0.2, 1.5), (0.05, 0.35, 0.14, 0.25)):
        img[((x - cx * rx) / rx) ** 2 + ((y - cy * ry) / ry) ** 2 <= rad**2] = val
    support = img > 0
    out = img.astype(complex)
    if smooth_phase:
        out = out * np.exp(1j * np.pi * (x / rx + 0.5 * y / ry))
    return out, support


def synth_coils(grid: Grid, n_coils: int, decay=0.6):
    """Gaussian-bump coil maps with linear phase ramps (nfs/simulate.py:123-142)."""
    c = grid_coordinates(grid)
    x, y = c[:, 0], c[:, 1]
    rx, ry = grid.fov_m[0] / 2, grid.fov_m[1] / 2
    w = decay * min(rx, ry)
    maps = np.zeros((grid.nvox, n_coils), complex)
    for lam in range(n_coils):
        th = 2 * np.pi * lam / n_coils
        cx, cy = 1.1 * rx * np.cos(th), 1.1 * ry * np.sin(th)
        mag = np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * w**2))
        ramp = np.pi * (np.cos(th) * x / rx + np.sin(th) * y / ry) * (0.5 + 0.1 * lam)
        maps[:, lam] = mag * np.exp(1j * ramp)
    return maps


def make_b0(grid: Grid, pattern="linear", amplitude=200.0):
    """Off-resonance map in rad/s (nfs/simulate.py:145-158)."""
    c = grid_coordinates(grid)
    if pattern == "zero":
        return np.zeros(grid.nvox)
    if pattern == "linear":
        return amplitude * c[:, 0] / (grid.fov_m[0] / 2)
    raise ValueError(pattern)


def higher_order_terms(t, n_extra, k_nyq, half_fov, scale=0.05):
    """Synthetic higher-order field time courses (nfs/pipeline.py:82-97)."""
    t_end = t[-1] if t[-1] > 0 else 1.0
    cols = [scale * k_nyq / half_fov ** (1 if p < 5 else 2) * np.sin(2 * np.pi * (p + 1) * t / t_end)
            for p in range(n_extra)]
    return np.column_stack(cols)


@dataclass
class Problem:
    """One synthetic reconstruction problem (inputs of EncodingInputs minus sigma)."""

    name: str
    grid: Grid
    spatial: np.ndarray     # (P+1, L_R)
    temporal: np.ndarray    # (K, P+1)
    sens: np.ndarray        # (L_R, Gamma)
    intensity: np.ndarray   # (L_R,)
    mask_r: np.ndarray      # (L,)
    rho_true: np.ndarray    # (L_R,) restricted ground truth
    n_iter: int


def _bases(grid, b0, mask, traj, order, z_offset=0.0):
    """Spatial/temporal tables; order > 1 appends synthetic higher-order terms.  `z_offset`
    moves a 2D slice off the isocentre (config C): the harmonics are evaluated at z = z_offset."""
    nd = grid.ndim
    coords = grid_coordinates(grid)[mask]
    if z_offset:
        coords = coords.copy()
        coords[:, 2] += z_offset
    harm = solid_harmonics(order, coords, ndim=nd)
    terms = traj[:, 1:]
    if harm.shape[1] > terms.shape[1]:
        k_nyq = np.pi * min(n / f for n, f in zip(grid.dims[:nd], grid.fov_m[:nd]))
        extra = higher_order_terms(traj[:, 0], harm.shape[1] - terms.shape[1], k_nyq,
                                   min(grid.fov_m[:nd]) / 2)
        terms = np.column_stack([terms, extra])
    spatial = np.vstack([b0[mask][None, :], harm.T])
    temporal = np.column_stack([traj[:, 0], terms])
    return spatial, temporal


def make_problem(name: str, scale: int = 1) -> Problem:
    """Configs of SURVEY.md 8d.  `scale` > 1 shrinks B/D in-plane for parity runs.

    A: 64x64, 8 coils, K=16384 spiral, B0 + linear terms (P+1=3), 20 iterations.
    A_mask: A restricted to the phantom support with intensity correction.
    B: 256x256 disc mask r<=0.45 FOV, 32 coils, K=65536 over 71.5 ms, B0 + 15 third-order
       harmonic terms (P+1=16), 20 iterations.
    D: 128x128x64 stack of 64 spirals x 4682 samples, 32 coils, B0 + 15 terms, 50 it.
    """
    if name in ("A", "A_mask"):
        grid = Grid((64, 64, 1), (0.22, 0.22, 0.002))
        traj = make_spiral(16384, turns=32, k_max=np.pi * 64 / 0.22, readout_s=0.03)
        n_coils, order, n_iter = 8, 1, 20
        rho, support = make_phantom(grid, "discs", smooth_phase=True)
        mask = support if name == "A_mask" else np.ones(grid.nvox, bool)
    elif name == "B":
        n = 256 // scale
        grid = Grid((n, n, 1), (0.22, 0.22, 0.002))
        traj = make_spiral(65536 // scale**2, turns=32 / scale, k_max=np.pi * n / 0.22,
                           readout_s=0.0715)
        n_coils, order, n_iter = 32, 3, 20
        rho, _ = make_phantom(grid, "discs", smooth_phase=True)
        c = grid_coordinates(grid)
        mask = np.hypot(c[:, 0], c[:, 1]) <= 0.45 * 0.22
    elif name == "D":
        nxy, nz = 128 // scale, 64 // scale
        grid = Grid((nxy, nxy, nz), (0.22, 0.22, 0.128))
        per_plane = 4682 // scale**2
        traj = make_spiral(per_plane, turns=9.14 / scale, k_max=np.pi * nxy / 0.22,
                           readout_s=0.03, ndim=3, n_planes=nz, kz_max=np.pi * nz / 0.128)
        n_coils, order, n_iter = 32, 3, 50
        rho, _ = make_phantom(grid, "discs", smooth_phase=True)
        c = grid_coordinates(grid)
        # ellipsoid with ~50 % of the volume
        mask = (c[:, 0] / 0.11) ** 2 + (c[:, 1] / 0.11) ** 2 + (c[:, 2] / 0.064) ** 2 <= 0.98
    else:
        raise ValueError(f"unknown config {name!r}")
    b0 = make_b0(grid, "linear", 200.0)
    spatial, temporal = _bases(grid, b0, mask, traj, order)
    sens_full = synth_coils(grid, n_coils)
    if name == "A":
        intensity = np.ones(int(mask.sum()))
    else:
        ssq = (np.abs(sens_full) ** 2).sum(axis=1)
        intensity = 1.0 / np.sqrt(ssq[mask])
    return Problem(name, grid, spatial, temporal, sens_full[mask], intensity, mask,
                   rho[mask], n_iter)


def slice_offsets(n_slices: int = 40, spacing_m: float = 0.002) -> np.ndarray:
    """Slice centres of a multi-slice stack, symmetric about the isocentre (config C)."""
    return spacing_m * (np.arange(n_slices) - (n_slices - 1) / 2.0)


def make_slices(n_slices: int = 40, spacing_m: float = 0.002, scale: int = 1, which=None):
    """Config C: a stack of `n_slices` config-B slices at z offsets +-, 2 mm apart,
    sharing the trajectory and its field-term time courses; each slice's spatial basis holds
    the third-order solid harmonics at ITS z (z != 0 switches on the z-dependent terms).
    Every slice is an independent reconstruction problem (replicas across GPUs, no
    collective).  `which` selects slice indices (default all)."""
    base = make_problem("B", scale=scale)
    n = 256 // scale
    grid = base.grid
    traj = make_spiral(65536 // scale**2, turns=32 / scale, k_max=np.pi * n / 0.22, readout_s=0.0715)
    b0 = make_b0(grid, "linear", 200.0)
    out = []
    zs = slice_offsets(n_slices, spacing_m)
    for i in (range(n_slices) if which is None else which):
        spatial, temporal = _bases(grid, b0, base.mask_r, traj, 3, z_offset=float(zs[i]))
        rho = base.rho_true * (0.75 + 0.5 * i / max(n_slices - 1, 1))   # slice-dependent contrast
        out.append(Problem(f"C[{i}] z={zs[i] * 1e3:+.1f} mm", grid, spatial, temporal, base.sens,
                           base.intensity, base.mask_r, rho, base.n_iter))
    return out
