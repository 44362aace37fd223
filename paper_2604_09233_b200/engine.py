"""Drop-in GPU engine: the reference's engine API on the B200 path.

Same names, signatures, argument meaning, exception classes and CGLog contents as the
reference's `nfs/engine.py` (cited per function).  Every numeric operation on the hot path
runs in the CUDA extension (`_nfs_b200.so`, include/nfs_b200.h) -- there is no CPU fallback.

Precision: the operators run in FP64 parity mode by default ("fp64": FP64 phase, sincospi
and FMA), which reproduces the reference's own 1e-10/1e-12 tests.  The fast modes are
selected per call (`precision="fp32"` or `"tf32x3"`) or process-wide via the environment
variable NFS_B200_PRECISION.  DESIGN.md states the tolerance of each mode.

Multi-GPU: when torch.distributed is initialised with world_size > 1, `recon_full` /
`recon_split` shard the readout samples across ranks (contiguous rows) and all-reduce the
adjoint image once per iteration over NCCL; every rank returns the result.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .core import Grid, ReconImage, grid_coordinates
from .errors import EngineError, MemoryBudgetError
from .simulate import solid_harmonics

__all__ = [
    "EngineError", "MemoryBudgetError", "EncodingInputs", "CGLog", "phase_block", "apply_E",
    "apply_EH", "recon_full", "recon_split", "choose_block_starts", "build_bases",
    "default_precision", "PhaseBlock", "DeviceSens", "DatasetSamples", "intensity_correction",
]


def default_precision() -> str:
    return os.environ.get("NFS_B200_PRECISION", "fp64")


def default_device() -> int:
    env = os.environ.get("NFS_B200_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------------------------
# types (nfs/engine.py:30-90)
# ----------------------------------------------------------------------------------

@dataclass
class EncodingInputs:
    """Inputs of the reconstruction, voxel arrays restricted to the mask (nfs/engine.py:30-78)."""

    sigma: np.ndarray
    spatial: np.ndarray
    temporal: np.ndarray
    sens: np.ndarray
    intensity: np.ndarray
    kfilter: np.ndarray | None
    mask_r: np.ndarray
    grid: Grid
    n_iter: int
    block_starts: np.ndarray | None = None

    def __post_init__(self):
        k, gam = self.sigma.shape
        p1, l_r = self.spatial.shape
        if self.temporal.shape != (k, p1):
            raise EngineError(
                f"temporal basis shape {self.temporal.shape} does not match samples {k} / terms {p1}")
        if self.sens.shape != (l_r, gam):
            raise EngineError(
                f"sensitivity shape {self.sens.shape} does not match voxels {l_r} / coils {gam}")
        if self.intensity.shape != (l_r,):
            raise EngineError("intensity correction length mismatch")
        self.mask_r = np.asarray(self.mask_r, dtype=bool).reshape(-1)
        if int(self.mask_r.sum()) != l_r:
            raise EngineError("reconstruction mask does not match restricted arrays")
        if self.block_starts is not None:
            ks = np.asarray(self.block_starts, dtype=int)
            if ks[0] != 0 or ks[-1] != k or np.any(np.diff(ks) <= 0):
                raise EngineError("block starts must increase from 0 to the sample count")
            self.block_starts = ks

    @property
    def n_samples(self) -> int:
        return self.sigma.shape[0]

    @property
    def n_voxels(self) -> int:
        return self.spatial.shape[1]


@dataclass
class CGLog:
    """Per-iteration norms and per-phase timings (nfs/engine.py:81-90)."""

    residual_norms: list = field(default_factory=list)
    solution_norms: list = field(default_factory=list)
    timings: list = field(default_factory=list)

    def add_timing(self, label: str, seconds: float):
        self.timings.append((label, seconds))


# ----------------------------------------------------------------------------------
# lazy phase handle (nfs/engine.py:93-95)
# ----------------------------------------------------------------------------------

class DeviceSpatial:
    """Spatial basis (P+1, L_R) described by the grid, mask, B0 map and harmonic order; the
    table is evaluated on the GPU by `nfs_set_tables_grid`, so only a voxel index
    and B0 per voxel cross PCIe.  `np.asarray(handle)` builds the identical host table with the
    reference formulas (nfs/engine.py:252-280), so it can stand in for the array anywhere.
    """

    __array_priority__ = 10

    def __init__(self, b0, mask_r, grid: Grid, order: int):
        self.mask_r = np.asarray(mask_r, dtype=bool).reshape(-1)
        self.b0 = np.asarray(b0, dtype=float).reshape(-1)
        if self.b0.size != self.mask_r.size or self.mask_r.size != grid.nvox:
            raise EngineError("B0 map and mask must cover the grid")
        if order not in (1, 2, 3):
            raise EngineError(f"unsupported harmonic order {order}")
        self.grid, self.order = grid, int(order)
        self.vox_index = np.flatnonzero(self.mask_r).astype(np.int64)
        self.b0_masked = np.ascontiguousarray(self.b0[self.mask_r])
        n_h = {1: 2 if grid.ndim == 2 else 3, 2: 8, 3: 15}[self.order]
        self.shape = (1 + n_h, int(self.vox_index.size))

    @property
    def dtype(self):
        return np.dtype(np.float64)

    def __array__(self, dtype=None, copy=None):
        coords = grid_coordinates(self.grid)[self.mask_r]
        harm = solid_harmonics(self.order, coords, ndim=self.grid.ndim)
        arr = np.vstack([self.b0_masked[None, :], harm.T])
        return arr if dtype is None else arr.astype(dtype)

    def upload(self, plan, temporal):
        plan.set_tables_grid(temporal, self.vox_index, self.b0_masked, self.grid.dims, self.grid.fov_m, self.order)


class DeviceRMSE:
    """Convergence-study callback computed on the GPU.

    Equivalent to the reference pattern (tests/test_acceptance.py:346-375)::

        def cb(n, rho_r):
            full = zeros(L); full[mask_r] = rho_r * j; errs.append(metrics.rmse(full, ref, support))

    Passed as `callback=` to recon_full / recon_split (alone or in a list with DeviceSSIM), the
    relative RMSE of every iterate is evaluated inside the device CG loop (no per-iteration host
    copy of the iterate) and lands in `.values` when the solve returns.
    """

    def __init__(self, reference, support=None):
        self.reference = np.asarray(reference).reshape(-1)
        self.support = None if support is None else np.asarray(support, dtype=bool).reshape(-1)
        self.values: list = []

    def _restricted(self, mask_r, intensity):
        sup = np.ones(self.reference.size, bool) if self.support is None else self.support
        if sup.size != mask_r.size or self.reference.size != mask_r.size:
            raise EngineError("RMSE reference / support must cover the grid")
        ref_sq = float(np.sum(np.abs(self.reference[sup]) ** 2))
        if ref_sq == 0.0:
            raise EngineError("reference is zero on the mask")
        on = sup[mask_r]
        ref_m = np.where(on, self.reference[mask_r], 0.0).astype(np.complex128)
        w = np.where(on, np.asarray(intensity, dtype=float), 0.0)
        outside = float(np.sum(np.abs(self.reference[sup & ~mask_r]) ** 2))
        return ref_m, w, outside, ref_sq

    def _attach(self, plan, inputs):
        plan.set_rmse_reference(*self._restricted(inputs.mask_r, inputs.intensity))

    def _collect(self, plan, n_done):
        self.values = plan.rmse_log(n_done)
        plan.set_rmse_reference(None, None, 0.0, 0.0)

    def __call__(self, n, rho_r):
        raise EngineError("DeviceRMSE is evaluated on the device by recon_full / recon_split")


class DeviceSSIM:
    """Per-iteration mean SSIM of the magnitude image on the GPU.

    Equivalent to a convergence-study callback computing
    ``metrics.ssim(abs(full).reshape(nx, ny, order="F"), reference, window, sigma, k1, k2, mask)``
    (nfs/metrics.py:20-70) with ``full[mask_r] = rho_r * j`` on a 2D grid; the values land in
    `.values` when the solve returns.
    """

    def __init__(self, reference, window: int = 11, sigma: float = 1.5, k1: float = 0.01, k2: float = 0.03,
                 mask=None):
        self.reference = np.asarray(reference, dtype=float)
        if self.reference.ndim != 2:
            raise EngineError("ssim expects a 2D reference image (nx, ny)")
        nx, ny = self.reference.shape
        if nx < window or ny < window:
            raise EngineError(f"image smaller than the {window}x{window} window")
        drange = float(self.reference.max() - self.reference.min())
        if drange == 0:
            raise EngineError("reference image is constant")
        half = (window - 1) / 2.0
        ax = np.arange(window) - half
        g = np.exp(-(ax ** 2) / (2 * sigma ** 2))
        kern = np.outer(g, g)
        self.kern = kern / kern.sum()
        self.window, self.c1, self.c2 = int(window), (k1 * drange) ** 2, (k2 * drange) ** 2
        self.sel = None
        if mask is not None:
            m = np.asarray(mask, dtype=bool).reshape(nx, ny)
        h = (window - 1) // 2
        if mask is not None:
            sel = m[h:h + nx - window + 1, h:h + ny - window + 1]
            if not sel.any():
                raise EngineError("mask covers no valid windows")
            self.sel = sel.reshape(-1, order="F").astype(np.uint8)
        self.values: list = []

    def _attach(self, plan, inputs):
        grid = inputs.grid
        nx, ny = self.reference.shape
        if grid.dims[2] != 1 or (grid.dims[0], grid.dims[1]) != (nx, ny):
            raise EngineError("SSIM reference must match the 2D grid")
        vox = np.flatnonzero(inputs.mask_r).astype(np.int64)
        plan.set_ssim_reference(vox, np.asarray(inputs.intensity, dtype=float), nx, ny,
                                self.reference.reshape(-1, order="F"), self.kern, self.c1, self.c2, self.sel)

    def _collect(self, plan, n_done):
        self.values = plan.ssim_log(n_done)
        plan.set_ssim_reference(None, None, 0, 0, None, None, 0.0, 0.0)

    def __call__(self, n, rho_r):
        raise EngineError("DeviceSSIM is evaluated on the device by recon_full / recon_split")


_DEVICE_DIAGNOSTICS = (DeviceRMSE, DeviceSSIM)


class PhaseBlock:
    """P' = exp(i * temporal_rows @ spatial), never materialised on the hot path.

    Holds the basis tables; `apply_E` / `apply_EH` regenerate the phasors on the device.
    `np.asarray(handle)` materialises the block on the GPU (FP64 unless `precision` says
    otherwise) for small sizes, so code that inspects the matrix keeps working.
    """

    __array_priority__ = 10

    def __init__(self, temporal_rows, spatial, precision=None, device=None):
        self.temporal = np.ascontiguousarray(temporal_rows, dtype=np.float64)
        self.spatial = np.ascontiguousarray(spatial, dtype=np.float64)
        if self.temporal.ndim != 2 or self.spatial.ndim != 2 or \
                self.temporal.shape[1] != self.spatial.shape[0]:
            raise EngineError("temporal rows and spatial basis shapes do not match")
        self.precision = precision or default_precision()
        self.device = default_device() if device is None else device
        self._plans = {}

    @property
    def shape(self):
        return (self.temporal.shape[0], self.spatial.shape[1])

    @property
    def dtype(self):
        return np.dtype(np.complex128)

    def plan(self, n_coils: int) -> _native.Plan:
        key = (int(n_coils), self.precision)
        plan = self._plans.get(key)
        if plan is None:
            k, l = self.shape
            plan = _native.Plan(k, l, n_coils, self.temporal.shape[1], self.precision, self.device)
            plan.set_tables(self.temporal, self.spatial)
            self._plans[key] = plan
        return plan

    def materialize(self) -> np.ndarray:
        k, _ = self.shape
        return self.plan(1).phase_rows(0, k)

    def __array__(self, dtype=None, copy=None):
        out = self.materialize()
        return out if dtype is None else out.astype(dtype)

    def __abs__(self):
        return np.abs(self.materialize())


class DeviceSens:
    """Full-grid coil maps plus the reconstruction mask, standing in for the restricted maps
    `sens_full[mask_r]` of EncodingInputs.sens: the mask restriction and S' = S o j
    run on the GPU at upload (`nfs_set_sens_grid`), and `.intensity` is the intensity correction
    j = 1/sqrt(sum_c |S|^2) of the reconstructed voxels computed on the GPU
    (nfs/sensmaps.py:145-152, restricted as nfs/pipeline.py:203).  `np.asarray(handle)` gives the
    host restriction, so the handle can stand in for the array anywhere."""

    __array_priority__ = 10

    def __init__(self, sens_full, mask_r, device: int | None = None):
        self.sens_full = np.ascontiguousarray(sens_full, dtype=np.complex128)
        self.mask_r = np.asarray(mask_r, dtype=bool).reshape(-1)
        if self.sens_full.ndim != 2 or self.sens_full.shape[0] != self.mask_r.size:
            raise EngineError("full-grid sensitivities and mask do not match")
        self.vox_index = np.flatnonzero(self.mask_r).astype(np.int64)
        self.device = default_device() if device is None else device
        self._j = None

    @property
    def shape(self):
        return (int(self.vox_index.size), int(self.sens_full.shape[1]))

    @property
    def ndim(self):
        return 2

    @property
    def dtype(self):
        return np.dtype(np.complex128)

    def __array__(self, dtype=None, copy=None):
        out = self.sens_full[self.mask_r]
        return out if dtype is None else out.astype(dtype)

    @property
    def intensity(self) -> np.ndarray:
        """j on the reconstructed voxels, evaluated on the GPU (cached)."""
        if self._j is None:
            self._j = _native.intensity_correction(self.sens_full, self.vox_index, self.device)
        return self._j


class DatasetSamples:
    """The raw coil samples of a reference dataset directory, left on disk: the
    reference stores them as `sigma.c128`, raw little-endian complex128 (K, coils) listed in
    `manifest.json` (nfs/core.py:292-328).  Used as EncodingInputs.sigma, each rank's plan reads
    ONLY its own sample rows from the file through the pinned staging ring
    (`nfs_set_samples_file`); `np.asarray(handle)` loads the whole array like
    `Dataset.load_array`.  Accepts a dataset directory or an nfsense `Dataset`."""

    __array_priority__ = 10

    def __init__(self, dataset, name: str = "sigma"):
        import json
        root = getattr(dataset, "path", dataset)
        root = os.fspath(root)
        with open(os.path.join(root, "manifest.json"), encoding="utf-8") as fh:
            entry = json.load(fh).get("arrays", {}).get(name)
        if entry is None:
            raise EngineError(f"dataset has no array {name!r}")
        if entry["dtype"] != "c128" or len(entry["shape"]) != 2:
            raise EngineError(f"array {name!r} is not a (samples, coils) complex128 array")
        self.path = os.path.join(root, entry["file"])
        self._shape = (int(entry["shape"][0]), int(entry["shape"][1]))
        if os.path.getsize(self.path) != self._shape[0] * self._shape[1] * 16:
            raise EngineError(f"array {name!r}: file size does not match its shape")

    @property
    def shape(self):
        return self._shape

    @property
    def ndim(self):
        return 2

    @property
    def dtype(self):
        return np.dtype(np.complex128)

    def __array__(self, dtype=None, copy=None):
        out = np.fromfile(self.path, dtype="<c16").reshape(self._shape)
        return out if dtype is None else out.astype(dtype)


def intensity_correction(maps: np.ndarray, mask_r) -> np.ndarray:
    """nfs/sensmaps.py:145-152 on the GPU: j = 1/sqrt(sum_coils |S|^2) on the mask, else 0."""
    mask_r = np.asarray(mask_r, dtype=bool).reshape(-1)
    j = np.zeros(np.asarray(maps).shape[0])
    j[mask_r] = _native.intensity_correction(maps, np.flatnonzero(mask_r), default_device())
    return j


def phase_block(temporal_rows: np.ndarray, spatial: np.ndarray) -> PhaseBlock:
    """Lazy device phase block for a row range (nfs/engine.py:93-95)."""
    return PhaseBlock(temporal_rows, spatial)


def _as_phase(phase) -> PhaseBlock:
    if isinstance(phase, PhaseBlock):
        return phase
    raise EngineError("phase must be the handle returned by phase_block(); "
                      "materialised phase matrices are not used on the GPU path")


def apply_E(p: np.ndarray, sens: np.ndarray, phase) -> np.ndarray:
    """Predicted coil samples P @ (S * p), shape (K, Gamma) (nfs/engine.py:98-100)."""
    ph = _as_phase(phase)
    sens = np.asarray(sens)
    plan = ph.plan(sens.shape[1])
    plan.set_sens(sens)
    return plan.apply_E(np.asarray(p).reshape(-1))


def apply_EH(sigma: np.ndarray, sens: np.ndarray, phase) -> np.ndarray:
    """Adjoint image sum_c conj(S) * (P^H sigma), shape (L_R,) (nfs/engine.py:103-108)."""
    ph = _as_phase(phase)
    sens = np.asarray(sens)
    plan = ph.plan(sens.shape[1])
    plan.set_sens(sens)
    return plan.apply_EH(np.asarray(sigma))


# ----------------------------------------------------------------------------------
# reconstruction drivers
# ----------------------------------------------------------------------------------

# Result classes: ours by default; `dispatch.install()` swaps in the reference's ReconImage /
# CGLog so callers of the reference API get the reference's own types back.
RESULT_TYPES = {"ReconImage": ReconImage, "CGLog": CGLog}


def _n_samples(inputs) -> int:   # duck-typed: the reference's EncodingInputs has no properties
    return int(inputs.sigma.shape[0])


def _n_voxels(inputs) -> int:
    return int(inputs.spatial.shape[1])


def _dist_info():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return dist, dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return None, 0, 1


def shard_rows(n_samples: int, rank: int, world: int):
    """Contiguous, balanced sample-row shard of `rank`."""
    base, extra = divmod(n_samples, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _nccl_unique_id(dist, rank):
    """Rank 0 creates an NCCL unique id (via torch's bundled NCCL) and broadcasts it."""
    import torch
    if torch.cuda.is_available():   # torch's NCCL collectives act on its current device
        torch.cuda.set_device(default_device())
    obj = [None]
    if rank == 0:
        import torch.cuda.nccl as tnccl
        obj[0] = bytes(tnccl.unique_id())
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


_COMMS = {}


def _shared_comm(dist, rank, world, device):
    """The process's NCCL communicator for (rank, world, device): created once (one unique-id
    broadcast), then borrowed by every plan, so repeated recons skip ncclCommInitRank."""
    key = (rank, world, device)
    comm = _COMMS.get(key)
    if comm is None:
        comm = _native.SharedComm(_nccl_unique_id(dist, rank), rank, world, device)
        _COMMS[key] = comm
    return comm


def _upload_agreed(dist, upload):
    """Run `upload` (a per-rank check happens inside); with several ranks, every rank learns
    whether any rank failed before the first collective of the solve, so none is left blocked."""
    err = None
    try:
        upload()
    except EngineError as exc:
        err = exc
    if dist is not None:
        import torch
        flag = torch.tensor([0 if err is None else 1], dtype=torch.int32,
                            device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(flag)
        if err is None and int(flag.item()) > 0:
            err = EngineError("raw data contains non-finite values (on another rank)")
    if err is not None:
        raise err


def _make_plan(inputs: EncodingInputs, precision: str, log: CGLog, timing_label: bool, shard: bool = True):
    """Create the device plan for this rank's sample shard; upload tables, S', sigma.

    `shard=False` solves the whole problem on this rank (independent slices, recon_slices)."""
    dist, rank, world = _dist_info() if shard else (None, 0, 1)
    lo, hi = shard_rows(_n_samples(inputs), rank, world)
    device = default_device()
    t0 = time.perf_counter()
    plan = _native.Plan(hi - lo, _n_voxels(inputs), inputs.sens.shape[1],
                        inputs.spatial.shape[0], precision, device)
    try:
        if world > 1:
            plan.use_comm(_shared_comm(dist, rank, world, device))
        t_plan = time.perf_counter() - t0
        t0 = time.perf_counter()
        if isinstance(inputs.sens, DeviceSens):              # restriction + S' = S o j on the GPU
            plan.set_sens_grid(inputs.sens.sens_full, inputs.sens.vox_index, inputs.intensity)
        else:
            plan.set_sens(inputs.sens, inputs.intensity)      # S' = S o j on upload
        log.add_timing("intensity_correction", time.perf_counter() - t0)
        t0 = time.perf_counter()
        if isinstance(inputs.spatial, DeviceSpatial):
            inputs.spatial.upload(plan, inputs.temporal[lo:hi])
        else:
            plan.set_tables(inputs.temporal[lo:hi], inputs.spatial)
        if timing_label:   # the GPU analogue of building P: plan + table upload
            log.add_timing("build_phase_matrix", t_plan + time.perf_counter() - t0)
        if isinstance(inputs.sigma, DatasetSamples):   # this rank's rows straight from the file
            _upload_agreed(dist if world > 1 else None, lambda: plan.set_samples_file(inputs.sigma.path, lo))
        else:
            plan.set_samples(inputs.sigma[lo:hi])   # raw data finiteness checked on the device
    except BaseException:
        plan.close()
        raise
    return plan


def _device_diagnostics(callback):
    """The device-evaluated diagnostics in `callback` (one object or a list), else ()."""
    if isinstance(callback, _DEVICE_DIAGNOSTICS):
        return (callback,)
    if isinstance(callback, (list, tuple)) and callback and all(isinstance(c, _DEVICE_DIAGNOSTICS) for c in callback):
        return tuple(callback)
    return ()


def _run_cg(plan, inputs: EncodingInputs, log: CGLog, callback):
    diags = _device_diagnostics(callback)
    for d in diags:
        d._attach(plan, inputs)
    if diags:
        callback = None
    rho, res, sol, tim, n_done = plan.cg_solve(inputs.n_iter, callback)
    for d in diags:
        d._collect(plan, n_done)
    log.add_timing("initial_adjoint", float(tim[0]))
    for n in range(1, n_done + 1):
        log.add_timing(f"cg_iteration_{n}", float(tim[1 + n]))
    log.residual_norms.extend(res)
    log.solution_norms.extend(sol)
    return rho


def _finalize(rho_r: np.ndarray, inputs: EncodingInputs, log: CGLog) -> ReconImage:
    """rho o j, scatter to the grid, optional k-space filter (nfs/engine.py:111-122)."""
    from .kfilter import apply_filter

    t0 = time.perf_counter()
    full = np.zeros(inputs.mask_r.size, dtype=complex)
    full[inputs.mask_r] = rho_r * inputs.intensity
    log.add_timing("apply_intensity", time.perf_counter() - t0)
    if inputs.kfilter is not None:
        t0 = time.perf_counter()
        full = apply_filter(full, inputs.kfilter, inputs.grid, device=default_device())
        log.add_timing("apply_kfilter", time.perf_counter() - t0)
    res = log.residual_norms[-1] if log.residual_norms else 0.0
    return RESULT_TYPES["ReconImage"](values=full, iterations=inputs.n_iter, final_residual=res)


def recon_full(inputs: EncodingInputs, memory_budget_bytes: int | None = None, callback=None,
               *, precision: str | None = None):
    """CG reconstruction (nfs/engine.py:125-179).

    The phase matrix is never stored on the GPU; the reference's budget rule
    (K * L_R * 16 bytes > budget -> MemoryBudgetError) is kept because callers and the
    CLI exit codes depend on it.  `callback(n, rho_restricted)` runs after each iteration.
    """
    need = _n_samples(inputs) * _n_voxels(inputs) * 16
    if memory_budget_bytes is not None and need > memory_budget_bytes:
        raise MemoryBudgetError(
            f"phase matrix needs {need} bytes (> budget {memory_budget_bytes}); use the split variant")
    return _recon_full(inputs, callback, precision, shard=True)


def _check_samples(inputs: EncodingInputs, shard: bool):
    # single rank: nfs_set_samples checks finiteness on the device (same error); sharded: every
    # rank must fail together before any collective, so check the full array on the host
    if isinstance(inputs.sigma, DatasetSamples):   # checked per rank on upload (_upload_agreed)
        return
    if shard and _dist_info()[2] > 1 and not np.all(np.isfinite(inputs.sigma)):
        raise EngineError("raw data contains non-finite values")


def _recon_full(inputs: EncodingInputs, callback, precision, shard: bool):
    log = RESULT_TYPES["CGLog"]()
    _check_samples(inputs, shard)
    plan = _make_plan(inputs, precision or default_precision(), log, timing_label=True, shard=shard)
    try:
        rho = _run_cg(plan, inputs, log, callback)
    finally:
        plan.close()
    return _finalize(rho, inputs, log), log


def recon_slices(inputs_list, memory_budget_bytes: int | None = None, *, precision: str | None = None,
                 gather: bool = True):
    """Independent problems (slices of a multi-slice acquisition).

    With torch.distributed initialised, slice i is reconstructed by rank i mod world with no
    collective in the solve ("replicas" of the solver, not of the data); `gather=True` returns
    every slice's (ReconImage, CGLog) on every rank (one all_gather of the results), otherwise
    each rank gets only its own slices (None elsewhere).  Each slice follows recon_full's rules.
    """
    dist, rank, world = _dist_info()
    out = [None] * len(inputs_list)
    failures = {}
    for i, inputs in enumerate(inputs_list):
        if i % world != rank:
            continue
        try:
            need = _n_samples(inputs) * _n_voxels(inputs) * 16
            if memory_budget_bytes is not None and need > memory_budget_bytes:
                raise MemoryBudgetError(
                    f"phase matrix needs {need} bytes (> budget {memory_budget_bytes}); use the split variant")
            out[i] = _recon_full(inputs, None, precision, shard=False)
        except Exception as exc:   # no rank may skip the gather below (it would deadlock the others)
            failures[i] = exc
            if world == 1:
                raise
    if world > 1:
        # every rank reaches this collective, failed or not; the first failure (lowest slice
        # index) is re-raised on every rank
        parts = [None] * world
        mine = {i: r for i, r in enumerate(out) if r is not None} if gather else {}
        dist.all_gather_object(parts, (mine, {i: (type(e), str(e)) for i, e in failures.items()}))
        errs = {}
        for part, fails in parts:
            errs.update(fails)
            for i, r in part.items():
                out[i] = r
        if errs:
            i = min(errs)
            if i in failures:
                raise failures[i]
            cls, msg = errs[i]
            raise (cls if isinstance(cls, type) and issubclass(cls, EngineError) else EngineError)(
                f"slice {i} failed on another rank: {msg}")
    return out


def recon_split(inputs: EncodingInputs, callback=None, *, precision: str | None = None):
    """Split-variant CG (nfs/engine.py:182-241).

    On the GPU both variants regenerate the phase on the fly, so the block structure only
    affects validation; results equal `recon_full` bit for bit.
    """
    if inputs.block_starts is None:
        raise EngineError("split reconstruction needs block starts")
    log = RESULT_TYPES["CGLog"]()
    _check_samples(inputs, True)
    plan = _make_plan(inputs, precision or default_precision(), log, timing_label=False)
    try:
        rho = _run_cg(plan, inputs, log, callback)
    finally:
        plan.close()
    return _finalize(rho, inputs, log), log


def choose_block_starts(n_samples: int, n_voxels: int, memory_budget_bytes: int) -> np.ndarray:
    """Largest row block whose c128 phase block fits the budget (nfs/engine.py:244-249)."""
    rows = max(1, min(n_samples, memory_budget_bytes // max(n_voxels * 16, 1)))
    return np.unique(np.asarray(list(range(0, n_samples, rows)) + [n_samples], dtype=int))


def build_bases(b0, mask_r, grid: Grid, times_s, field_terms, order: int = 1, *, on_device: bool = False):
    """Spatial (P+1, L_R) and temporal (K, P+1) basis tables (nfs/engine.py:252-280).

    `on_device=True` returns a `DeviceSpatial` handle instead of the spatial array: recon_full /
    recon_split then evaluate the table on the GPU; `np.asarray(handle)` gives the
    identical host array.
    """
    mask_r = np.asarray(mask_r, dtype=bool).reshape(-1)
    b0 = np.asarray(b0, dtype=float).reshape(-1)
    if on_device:
        spatial = DeviceSpatial(b0, mask_r, grid, order)   # table evaluated on the GPU at upload
        n_h = spatial.shape[0] - 1
    else:
        harm = solid_harmonics(order, grid_coordinates(grid)[mask_r], ndim=grid.ndim)
        spatial, n_h = None, harm.shape[1]
    field_terms = np.asarray(field_terms, dtype=float)
    if field_terms.ndim != 2 or field_terms.shape[1] != n_h:
        got = field_terms.shape[1] if field_terms.ndim == 2 else "?"
        raise EngineError(f"trajectory provides {got} field terms but order {order} needs {n_h}")
    times_s = np.asarray(times_s, dtype=float).reshape(-1)
    if times_s.size != field_terms.shape[0]:
        raise EngineError("sample time count does not match field terms")
    temporal = np.column_stack([times_s, field_terms])
    if spatial is None:
        spatial = np.vstack([b0[mask_r][None, :], harm.T])
    return spatial, temporal
