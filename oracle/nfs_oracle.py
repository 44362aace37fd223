"""CPU ORACLE — test infrastructure only, never shipped, never on the product path.

A plain-numpy restatement of the non-Fourier SENSE hot path of the reference package
(`/root/reference/pkg/src/nfsense`, abbreviated `nfs/` below).  Only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of `bench.py`
may import this module, and only as the checker / CPU baseline.

Parity is PINNED: `tests/test_oracle_golden.py` checks every function here against
golden vectors produced by importing the real reference in the build container
(`tests/golden/make_golden.py`), and the reference's own known-answer properties
(dense-matrix equivalence, adjoint identity, exact recovery, split == full).

Arithmetic lives in numpy ufuncs and OpenBLAS zgemm/dgemm exactly as in the reference
(`nfs/engine.py:95,100,108,206,222`); the reference pins only `numpy>=1.24`
(`pkg/pyproject.toml:10-15`).
"""

from __future__ import annotations

import time

import numpy as np


class OracleEngineError(Exception):
    """Mirrors nfs/engine.py:22 EngineError."""


class OracleMemoryBudgetError(OracleEngineError):
    """Mirrors nfs/engine.py:26 MemoryBudgetError (message mentions 'split')."""


# ----------------------------------------------------------------------------------
# geometry and bases
# ----------------------------------------------------------------------------------

def grid_coordinates(dims, fov_m) -> np.ndarray:
    """Voxel-centre coordinates (L, 3) in metres, x fastest.  nfs/core.py:102-113."""
    per_axis = [(f / n) * (np.arange(n) - 0.5 * (n - 1)) for n, f in zip(dims, fov_m)]
    gx, gy, gz = np.meshgrid(*per_axis, indexing="ij")
    return np.stack([a.reshape(-1, order="F") for a in (gx, gy, gz)], axis=1)


def solid_harmonics(order: int, coords: np.ndarray, ndim: int = 3,
                    include_constant: bool = False) -> np.ndarray:
    """Harmonic polynomial terms, nfs/simulate.py:26-59 (orders 1..3, 2/3/8/15 terms)."""
    if order not in (1, 2, 3):
        raise ValueError(order)
    x, y, z = (np.asarray(coords, float)[:, i] for i in range(3))
    cols = [np.ones_like(x)] if include_constant else []
    cols += [x, y] if (ndim == 2 and order == 1) else [x, y, z]
    if order >= 2:
        x2, y2, z2 = x * x, y * y, z * z
        cols += [x * y, z * y, 2 * z2 - x2 - y2, z * x, x2 - y2]
    if order >= 3:
        cols += [y * (3 * x2 - y2), x * y * z, y * (4 * z2 - x2 - y2),
                 z * (2 * z2 - 3 * x2 - 3 * y2), x * (4 * z2 - x2 - y2),
                 z * (x2 - y2), x * (x2 - 3 * y2)]
    return np.stack(cols, axis=1)


def build_bases(b0, mask_r, dims, fov_m, times_s, field_terms, order=1):
    """Spatial (P+1, L_R) and temporal (K, P+1) tables.  nfs/engine.py:252-280."""
    mask_r = np.asarray(mask_r, bool).reshape(-1)
    coords = grid_coordinates(dims, fov_m)[mask_r]
    ndim = 2 if dims[2] == 1 else 3
    harm = solid_harmonics(order, coords, ndim=ndim)
    field_terms = np.asarray(field_terms, float)
    if field_terms.ndim != 2 or field_terms.shape[1] != harm.shape[1]:
        raise OracleEngineError("field term count does not match harmonic order")
    times_s = np.asarray(times_s, float).reshape(-1)
    if times_s.size != field_terms.shape[0]:
        raise OracleEngineError("sample time count mismatch")
    spatial = np.concatenate([np.asarray(b0, float).reshape(-1)[mask_r][None], harm.T], 0)
    temporal = np.concatenate([times_s[:, None], field_terms], 1)
    return spatial, temporal


def intensity_correction(sens_full, mask_r):
    """j = 1/sqrt(sum_c |S|^2) on the support, else 0.  nfs/sensmaps.py:145-152."""
    mask_r = np.asarray(mask_r, bool).reshape(-1)
    ssq = (np.abs(sens_full) ** 2).sum(axis=1)
    out = np.zeros(sens_full.shape[0])
    keep = mask_r & (ssq > 0)
    out[keep] = 1.0 / np.sqrt(ssq[keep])
    return out


# ----------------------------------------------------------------------------------
# operators
# ----------------------------------------------------------------------------------

def phase_block(temporal_rows, spatial):
    """P' = exp(i K_rows R).  nfs/engine.py:93-95."""
    return np.exp(1j * (temporal_rows @ spatial))


def apply_E(p, sens, phase):
    """y = P (S o p), (K, Gamma).  nfs/engine.py:98-100."""
    return phase @ (sens * p[:, None])


def apply_EH(sigma, sens, phase):
    """q = conj(colsum((sigma^H P) o S^T)) -- P^H never formed.  nfs/engine.py:103-108."""
    acc = sigma.conj().T @ phase
    return np.conj((acc * sens.T).sum(axis=0))


def choose_block_starts(n_samples, n_voxels, memory_budget_bytes):
    """Row blocks whose c128 phase block fits the budget.  nfs/engine.py:244-249."""
    rows = max(1, min(n_samples, memory_budget_bytes // max(16 * n_voxels, 1)))
    return np.unique(np.asarray(list(range(0, n_samples, rows)) + [n_samples], dtype=int))


def forward_signal(rho, sens, spatial, temporal):
    """Sample-by-sample signal model (loop oracle).  nfs/simulate.py:219-244 (noise-free)."""
    rho = np.asarray(rho, complex).reshape(-1)
    out = np.empty((temporal.shape[0], sens.shape[1]), complex)
    for k in range(temporal.shape[0]):
        phi = np.zeros(rho.size)
        for p in range(temporal.shape[1]):
            phi = phi + temporal[k, p] * spatial[p]
        carrier = np.exp(1j * phi) * rho
        for c in range(sens.shape[1]):
            out[k, c] = np.sum(sens[:, c] * carrier)
    return out


def dense_encoding_matrix(sens, spatial, temporal):
    """Explicit E, rows coil-major (row = coil*K + sample).  nfs/simulate.py:247-262."""
    phi = np.zeros((temporal.shape[0], spatial.shape[1]))
    for p in range(temporal.shape[1]):
        phi += np.outer(temporal[:, p], spatial[p])
    carrier = np.exp(1j * phi)
    return np.concatenate([carrier * sens[:, c][None, :] for c in range(sens.shape[1])], 0)


# ----------------------------------------------------------------------------------
# CG drivers
# ----------------------------------------------------------------------------------

class OracleLog:
    """Mirrors nfs/engine.py:81-90 CGLog."""

    def __init__(self):
        self.residual_norms, self.solution_norms, self.timings = [], [], []


def _cg(p0, ehe, n_iter, log, callback):
    """Unpreconditioned CG on E^H E, exact reference update order.

    nfs/engine.py:154-178 (full) == :210-240 (split): early stop at the loop top when
    ||r|| <= 1e-15 ||r0||; complex step alpha/beta with beta = vdot(p, q); breakdown on
    beta == 0 or non-finite; non-finite iterate raises.
    """
    r = p0.copy()
    p = p0
    rho = np.zeros_like(p0)
    r0 = np.linalg.norm(r)
    for n in range(1, n_iter + 1):
        if np.linalg.norm(r) <= 1e-15 * r0:
            break
        t0 = time.perf_counter()
        q = ehe(p)
        alpha = np.vdot(r, r)
        beta = np.vdot(p, q)
        if beta == 0 or not np.isfinite(beta):
            raise OracleEngineError(f"CG breakdown at iteration {n}")
        step = alpha / beta
        rho = rho + step * p
        r = r - step * q
        beta = alpha
        alpha = np.vdot(r, r)
        p = r + (alpha / beta) * p
        log.timings.append((f"cg_iteration_{n}", time.perf_counter() - t0))
        if not np.all(np.isfinite(rho)):
            raise OracleEngineError(f"non-finite iterate at iteration {n}")
        log.residual_norms.append(float(np.sqrt(alpha.real)))
        log.solution_norms.append(float(np.linalg.norm(rho)))
        if callback is not None:
            callback(n, rho)
    return rho


def finalize(rho_r, intensity, mask_r, kfilter=None, dims=None):
    """rho o j, scatter to L, optional k-space filter.  nfs/engine.py:111-122."""
    full = np.zeros(np.asarray(mask_r).size, complex)
    full[np.asarray(mask_r, bool)] = rho_r * intensity
    if kfilter is not None:
        full = apply_filter(full, kfilter, dims)
    return full


def apply_filter(image, filt, dims):
    """IFFT(fftshift-centred FFT(image) * filter).  nfs/kfilter.py:83-97."""
    vol = np.asarray(image, complex).reshape(dims, order="F")
    spec = np.fft.fftshift(np.fft.fftn(vol)) * np.asarray(filt, float).reshape(dims, order="F")
    return np.fft.ifftn(np.fft.ifftshift(spec)).reshape(-1, order="F")


def recon_full(sigma, spatial, temporal, sens, intensity, n_iter, callback=None,
               memory_budget_bytes=None):
    """nfs/engine.py:125-179 minus finalisation; returns (rho_restricted, log)."""
    need = sigma.shape[0] * spatial.shape[1] * 16
    if memory_budget_bytes is not None and need > memory_budget_bytes:
        raise OracleMemoryBudgetError(f"phase matrix needs {need} bytes; use the split variant")
    if not np.all(np.isfinite(sigma)):
        raise OracleEngineError("raw data contains non-finite values")
    log = OracleLog()
    s_eff = sens * intensity[:, None]
    t0 = time.perf_counter()
    phase = phase_block(temporal, spatial)
    log.timings.append(("build_phase_matrix", time.perf_counter() - t0))
    t0 = time.perf_counter()
    p0 = apply_EH(sigma, s_eff, phase)
    log.timings.append(("initial_adjoint", time.perf_counter() - t0))
    rho = _cg(p0, lambda v: apply_EH(apply_E(v, s_eff, phase), s_eff, phase),
              n_iter, log, callback)
    return rho, log


def split_normal_apply(p, s_eff, spatial, temporal, starts):
    """One E^H E with per-block phase recompute.  nfs/engine.py:217-223."""
    w = s_eff * p[:, None]
    acc = np.zeros((s_eff.shape[1], s_eff.shape[0]), complex)
    for lo, hi in zip(starts[:-1], starts[1:]):
        blk = phase_block(temporal[lo:hi], spatial)
        acc += (blk @ w).conj().T @ blk
    return np.conj((acc * s_eff.T).sum(axis=0))


def split_adjoint(sigma, s_eff, spatial, temporal, starts):
    """Blockwise E^H sigma.  nfs/engine.py:199-207."""
    acc = np.zeros((s_eff.shape[1], s_eff.shape[0]), complex)
    sh = sigma.conj().T
    for lo, hi in zip(starts[:-1], starts[1:]):
        acc += sh[:, lo:hi] @ phase_block(temporal[lo:hi], spatial)
    return np.conj((acc * s_eff.T).sum(axis=0))


def recon_split(sigma, spatial, temporal, sens, intensity, n_iter, block_starts,
                callback=None):
    """nfs/engine.py:182-241 minus finalisation; returns (rho_restricted, log)."""
    if block_starts is None:
        raise OracleEngineError("split reconstruction needs block starts")
    if not np.all(np.isfinite(sigma)):
        raise OracleEngineError("raw data contains non-finite values")
    starts = np.asarray(block_starts, int)
    log = OracleLog()
    s_eff = sens * intensity[:, None]
    t0 = time.perf_counter()
    p0 = split_adjoint(sigma, s_eff, spatial, temporal, starts)
    log.timings.append(("initial_adjoint", time.perf_counter() - t0))
    rho = _cg(p0, lambda v: split_normal_apply(v, s_eff, spatial, temporal, starts),
              n_iter, log, callback)
    return rho, log


# ------------------------------------------------------------------ diagnostics
def gaussian_window(size=11, sigma=1.5):
    """Truncated, normalised 2D Gaussian window.  nfs/metrics.py:11-17."""
    half = (size - 1) / 2.0
    ax = np.arange(size) - half
    g = np.exp(-(ax ** 2) / (2 * sigma ** 2))
    k = np.outer(g, g)
    return k / k.sum()


def ssim(test, ref, window=11, sigma=1.5, k1=0.01, k2=0.03, mask=None):
    """Mean SSIM and map over all windows that fit; dynamic range from ref.  nfs/metrics.py:20-70
    (direct loops over window positions -- a restatement, not the sliding-window code)."""
    test, ref = np.asarray(test, float), np.asarray(ref, float)
    drange = float(ref.max() - ref.min())
    c1, c2 = (k1 * drange) ** 2, (k2 * drange) ** 2
    kern = gaussian_window(window, sigma)
    h0, w0 = test.shape[0] - window + 1, test.shape[1] - window + 1
    smap = np.empty((h0, w0))
    for i in range(h0):
        for j in range(w0):
            a, b = test[i:i + window, j:j + window], ref[i:i + window, j:j + window]
            mu1, mu2 = np.sum(kern * a), np.sum(kern * b)
            v1 = np.sum(kern * a * a) - mu1 ** 2
            v2 = np.sum(kern * b * b) - mu2 ** 2
            cov = np.sum(kern * a * b) - mu1 * mu2
            smap[i, j] = ((2 * mu1 * mu2 + c1) * (2 * cov + c2)) / ((mu1 ** 2 + mu2 ** 2 + c1) * (v1 + v2 + c2))
    if mask is not None:
        half = (window - 1) // 2
        sel = np.asarray(mask, bool)[half:half + h0, half:half + w0]
        return float(smap[sel].mean()), smap
    return float(smap.mean()), smap


def rmse(test, ref, mask=None):
    """||test - ref|| / ||ref|| (RMS) over the mask.  nfs/metrics.py:73-88."""
    test, ref = np.asarray(test).reshape(-1), np.asarray(ref).reshape(-1)
    if mask is not None:
        m = np.asarray(mask, bool).reshape(-1)
        test, ref = test[m], ref[m]
    return float(np.sqrt(np.mean(np.abs(test - ref) ** 2)) / np.sqrt(np.mean(np.abs(ref) ** 2)))
