"""ctypes binding of the C ABI in include/nfs_b200.h (the in-tree `_nfs_b200.so`).

There is no CPU fallback: if the shared library is missing or no CUDA device is visible,
every call raises `NativeUnavailable` (an EngineError).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError, EngineError, MemoryBudgetError, NativeUnavailable

LIB_PATH = os.environ.get("NFS_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_nfs_b200.so")

NFS_OK = 0
NFS_ERR_INVALID = 1
NFS_ERR_NONFINITE = 2
NFS_ERR_BREAKDOWN = 3
NFS_ERR_BUDGET = 4
NFS_ERR_CUDA = 5
NFS_ERR_NCCL = 6
NFS_ERR_NONFINITE_ITERATE = 7
NFS_ERR_ABORTED = 8

PRECISIONS = {"fp32": 0, "fp64": 1, "tf32x3": 2, "f16x3": 3}

_c_i32, _c_i64, _c_dbl_p, _c_void_p = ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
CALLBACK = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p)

# name -> (restype, argtypes); must match include/nfs_b200.h exactly
SIGNATURES = {
    "nfs_plan_create": (_c_i32, [ctypes.POINTER(_c_void_p), _c_i64, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32]),
    "nfs_plan_destroy": (None, [_c_void_p]),
    "nfs_plan_set_stream": (_c_i32, [_c_void_p, _c_void_p]),
    "nfs_plan_attach_comm": (_c_i32, [_c_void_p, ctypes.c_char_p, _c_i32, _c_i32]),
    "nfs_comm_create": (_c_i32, [ctypes.c_char_p, _c_i32, _c_i32, _c_i32, ctypes.POINTER(_c_void_p)]),
    "nfs_comm_destroy": (None, [_c_void_p]),
    "nfs_plan_use_comm": (_c_i32, [_c_void_p, _c_void_p, _c_i32, _c_i32]),
    "nfs_set_tables": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p]),
    "nfs_set_tables_t": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p]),
    "nfs_set_tables_grid": (_c_i32, [_c_void_p, _c_dbl_p, ctypes.POINTER(_c_i64), _c_dbl_p,
                                     ctypes.POINTER(_c_i32), _c_dbl_p, _c_i32]),
    "nfs_set_sens": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p]),
    "nfs_set_sens_grid": (_c_i32, [_c_void_p, _c_dbl_p, _c_i64, ctypes.POINTER(_c_i64), _c_dbl_p, _c_dbl_p]),
    "nfs_intensity_correction": (_c_i32, [_c_i32, _c_dbl_p, _c_i64, _c_i32, ctypes.POINTER(_c_i64), _c_i64,
                                          _c_dbl_p]),
    "nfs_set_samples": (_c_i32, [_c_void_p, _c_dbl_p]),
    "nfs_set_samples_file": (_c_i32, [_c_void_p, ctypes.c_char_p, _c_i64]),
    "nfs_apply_E": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p]),
    "nfs_apply_EH": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p]),
    "nfs_apply_EHE": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p]),
    "nfs_phase_rows": (_c_i32, [_c_void_p, _c_i64, _c_i64, _c_dbl_p]),
    "nfs_cg_solve": (_c_i32, [_c_void_p, _c_i32, CALLBACK, _c_void_p, _c_dbl_p, _c_dbl_p, _c_dbl_p,
                              ctypes.POINTER(_c_i32), _c_dbl_p]),
    "nfs_apply_EHE_resident": (_c_i32, [_c_void_p, _c_i32]),
    "nfs_set_rmse_reference": (_c_i32, [_c_void_p, _c_dbl_p, _c_dbl_p, ctypes.c_double, ctypes.c_double]),
    "nfs_rmse_log": (_c_i32, [_c_void_p, _c_dbl_p, _c_i32]),
    "nfs_set_ssim_reference": (_c_i32, [_c_void_p, ctypes.POINTER(_c_i64), _c_dbl_p, _c_i32, _c_i32, _c_dbl_p,
                                        _c_dbl_p, _c_i32, ctypes.c_double, ctypes.c_double,
                                        ctypes.POINTER(ctypes.c_uint8)]),
    "nfs_ssim_log": (_c_i32, [_c_void_p, _c_dbl_p, _c_i32]),
    "nfs_kernel_times": (_c_i32, [_c_void_p, _c_i32, ctypes.POINTER(ctypes.c_float)]),
    "nfs_bench_applies": (_c_i32, [_c_void_p, _c_i32, _c_i64, ctypes.POINTER(ctypes.c_float),
                                   ctypes.POINTER(ctypes.c_float)]),
    "nfs_launches_per_apply": (_c_i32, [_c_void_p]),
    "nfs_plan_describe": (ctypes.c_char_p, [_c_void_p]),
    "nfs_last_error": (ctypes.c_char_p, []),
    "nfs_version": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load the shared library and bind every declared symbol (raises if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"CUDA extension {path} is missing; build it with "
                "`python -m paper_2604_09233_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_c_dbl_p)


def _c128(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.complex128)
    if shape is not None and out.shape != tuple(shape):
        out = out.reshape(shape)
    return out


def _check(status: int):
    if status == NFS_OK:
        return
    msg = (load_library().nfs_last_error() or b"").decode()
    if status == NFS_ERR_BUDGET:
        raise MemoryBudgetError(f"{msg}; device memory exhausted, use the split variant or more GPUs")
    if status in (NFS_ERR_CUDA, NFS_ERR_NCCL):
        raise DeviceError(msg)
    raise EngineError(msg)


class Plan:
    """One device plan (include/nfs_b200.h nfs_plan)."""

    def __init__(self, n_samples, n_voxels, n_coils, n_terms, precision="fp32", device=0):
        lib = load_library()
        if precision not in PRECISIONS:
            raise EngineError(f"unknown precision {precision!r}; choose from {sorted(PRECISIONS)}")
        self._lib = lib
        self.shape = (int(n_samples), int(n_voxels), int(n_coils), int(n_terms))
        self.precision = precision
        self.device = int(device)
        h = _c_void_p()
        _check(lib.nfs_plan_create(ctypes.byref(h), int(n_samples), int(n_voxels), int(n_coils),
                                   int(n_terms), PRECISIONS[precision], int(device)))
        self._h = h

    # -- lifecycle ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.nfs_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def describe(self) -> str:
        return self._lib.nfs_plan_describe(self._h).decode()

    def set_stream(self, stream_ptr: int):
        _check(self._lib.nfs_plan_set_stream(self._h, _c_void_p(stream_ptr)))

    def attach_comm(self, unique_id: bytes, rank: int, world: int):
        _check(self._lib.nfs_plan_attach_comm(self._h, unique_id, rank, world))

    def use_comm(self, comm: "SharedComm"):
        _check(self._lib.nfs_plan_use_comm(self._h, comm.handle, comm.rank, comm.world))

    # -- inputs ------------------------------------------------------------------
    def set_tables(self, temporal, spatial):
        k, l, _, p1 = self.shape
        t = np.ascontiguousarray(temporal, dtype=np.float64).reshape(k, p1)
        spatial = np.asarray(spatial)
        if (spatial.dtype == np.float64 and spatial.shape == (p1, l) and spatial.flags.f_contiguous
                and not spatial.flags.c_contiguous):
            # build_bases' vstack yields a Fortran-ordered table: upload it voxel-major as is
            _check(self._lib.nfs_set_tables_t(self._h, _dp(t), _dp(spatial.T)))
            return
        s = np.ascontiguousarray(spatial, dtype=np.float64).reshape(p1, l)
        _check(self._lib.nfs_set_tables(self._h, _dp(t), _dp(s)))

    def set_tables_grid(self, temporal, vox_index, b0_masked, dims, fov, order):
        """Spatial table evaluated on the device; see nfs_set_tables_grid."""
        k, l, _, p1 = self.shape
        t = np.ascontiguousarray(temporal, dtype=np.float64).reshape(k, p1)
        v = np.ascontiguousarray(vox_index, dtype=np.int64).reshape(l)
        b = np.ascontiguousarray(b0_masked, dtype=np.float64).reshape(l)
        d = np.ascontiguousarray(dims, dtype=np.int32).reshape(3)
        f = np.ascontiguousarray(fov, dtype=np.float64).reshape(3)
        _check(self._lib.nfs_set_tables_grid(self._h, _dp(t), v.ctypes.data_as(ctypes.POINTER(_c_i64)), _dp(b),
                                             d.ctypes.data_as(ctypes.POINTER(_c_i32)), _dp(f), int(order)))

    def set_sens(self, sens, intensity=None):
        _, l, g, _ = self.shape
        s = _c128(sens, (l, g))
        j = None if intensity is None else np.ascontiguousarray(intensity, dtype=np.float64).reshape(l)
        _check(self._lib.nfs_set_sens(self._h, _dp(s.view(np.float64)),
                                      None if j is None else _dp(j)))

    def set_sens_grid(self, sens_full, vox_index, intensity=None):
        """S' from the full-grid maps: restriction (and j when intensity is None) on the device.
        Returns the j the device used (L_R,)."""
        _, l, g, _ = self.shape
        full = _c128(sens_full)
        idx = np.ascontiguousarray(vox_index, dtype=np.int64)
        if full.ndim != 2 or full.shape[1] != g or idx.shape != (l,):
            raise EngineError("full-grid sensitivity / voxel index shapes do not match the plan")
        j_out = np.empty(l)
        jin = None if intensity is None else np.ascontiguousarray(intensity, dtype=np.float64)
        _check(self._lib.nfs_set_sens_grid(self._h, _dp(full.view(np.float64)), int(full.shape[0]),
                                           idx.ctypes.data_as(ctypes.POINTER(_c_i64)),
                                           None if jin is None else _dp(jin), _dp(j_out)))
        return j_out

    def set_samples_file(self, path: str, row0: int = 0):
        """Samples = rows [row0, row0 + n_samples) of a raw complex128 (K, coils) dataset file."""
        _check(self._lib.nfs_set_samples_file(self._h, os.fsencode(path), int(row0)))

    def set_samples(self, sigma):
        k, _, g, _ = self.shape
        s = _c128(sigma, (k, g))
        _check(self._lib.nfs_set_samples(self._h, _dp(s.view(np.float64))))

    # -- operators -----------------------------------------------------------------
    def apply_E(self, p):
        k, l, g, _ = self.shape
        pv = _c128(p, (l,))
        y = np.empty((k, g), np.complex128)
        _check(self._lib.nfs_apply_E(self._h, _dp(pv.view(np.float64)), _dp(y.view(np.float64))))
        return y

    def apply_EH(self, sigma):
        k, l, g, _ = self.shape
        s = _c128(sigma, (k, g))
        q = np.empty(l, np.complex128)
        _check(self._lib.nfs_apply_EH(self._h, _dp(s.view(np.float64)), _dp(q.view(np.float64))))
        return q

    def apply_EHE(self, p):
        _, l, _, _ = self.shape
        pv = _c128(p, (l,))
        q = np.empty(l, np.complex128)
        _check(self._lib.nfs_apply_EHE(self._h, _dp(pv.view(np.float64)), _dp(q.view(np.float64))))
        return q

    def phase_rows(self, lo, hi):
        _, l, _, _ = self.shape
        out = np.empty((hi - lo, l), np.complex128)
        _check(self._lib.nfs_phase_rows(self._h, int(lo), int(hi), _dp(out.view(np.float64))))
        return out

    def cg_solve(self, n_iter, callback=None):
        """Returns (rho, residual_norms, solution_norms, timings_s, n_done)."""
        _, l, _, _ = self.shape
        rho = np.empty(l, np.complex128)
        res = np.zeros(max(n_iter, 1))
        sol = np.zeros(max(n_iter, 1))
        tim = np.zeros(2 + max(n_iter, 0))
        done = _c_i32(0)
        err = []

        def _cb(n, ptr, _user):
            try:
                arr = np.ctypeslib.as_array(ptr, shape=(2 * l,)).view(np.complex128).copy()
                callback(int(n), arr)
                return 0
            except BaseException as exc:  # abort the solve here, re-raise after the C call returns
                err.append(exc)
                return 1

        cfun = CALLBACK(_cb) if callback is not None else CALLBACK()
        status = self._lib.nfs_cg_solve(self._h, int(n_iter), cfun, None, _dp(rho.view(np.float64)),
                                        _dp(res), _dp(sol), ctypes.byref(done), _dp(tim))
        if err:
            raise err[0]
        _check(status)
        n = int(done.value)
        return rho, res[:n].tolist(), sol[:n].tolist(), tim, n

    def set_rmse_reference(self, ref_masked, weight, outside_sq, ref_sq):
        """Device per-iteration RMSE diagnostic; None switches it off."""
        _, l, _, _ = self.shape
        if ref_masked is None:
            _check(self._lib.nfs_set_rmse_reference(self._h, None, None, 0.0, 0.0))
            return
        r = _c128(ref_masked, (l,))
        w = np.ascontiguousarray(weight, dtype=np.float64).reshape(l)
        _check(self._lib.nfs_set_rmse_reference(self._h, _dp(r.view(np.float64)), _dp(w),
                                                float(outside_sq), float(ref_sq)))

    def set_ssim_reference(self, vox_index, weight, nx, ny, ref_img, kern, c1, c2, sel=None):
        """Device per-iteration SSIM diagnostic; ref_img None switches it off."""
        _, l, _, _ = self.shape
        if ref_img is None:
            _check(self._lib.nfs_set_ssim_reference(self._h, None, None, 0, 0, None, None, 0, 0.0, 0.0, None))
            return
        v = np.ascontiguousarray(vox_index, dtype=np.int64).reshape(l)
        w = np.ascontiguousarray(weight, dtype=np.float64).reshape(l)
        r = np.ascontiguousarray(ref_img, dtype=np.float64).reshape(-1)
        k = np.ascontiguousarray(kern, dtype=np.float64)
        sp = None
        if sel is not None:
            sel = np.ascontiguousarray(sel, dtype=np.uint8).reshape(-1)
            sp = sel.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        _check(self._lib.nfs_set_ssim_reference(self._h, v.ctypes.data_as(ctypes.POINTER(_c_i64)), _dp(w),
                                                int(nx), int(ny), _dp(r), _dp(k), int(k.shape[0]),
                                                float(c1), float(c2), sp))

    def ssim_log(self, n: int):
        out = np.zeros(max(int(n), 1))
        _check(self._lib.nfs_ssim_log(self._h, _dp(out), int(n)))
        return out[:int(n)].tolist()

    def rmse_log(self, n: int):
        out = np.zeros(max(int(n), 1))
        _check(self._lib.nfs_rmse_log(self._h, _dp(out), int(n)))
        return out[:int(n)].tolist()

    # -- benchmarking ------------------------------------------------------------------
    def apply_EHE_resident(self, n: int):
        _check(self._lib.nfs_apply_EHE_resident(self._h, int(n)))

    def kernel_times(self, reps: int = 3):
        out = (ctypes.c_float * 4)()
        _check(self._lib.nfs_kernel_times(self._h, int(reps), out))
        return list(out)

    def bench_applies(self, n: int, flush_bytes: int = 256 << 20):
        """(per-step ms list, summed forward / adjoint main-kernel ms) over n timed applies."""
        steps = (ctypes.c_float * max(int(n), 1))()
        kern = (ctypes.c_float * 2)()
        _check(self._lib.nfs_bench_applies(self._h, int(n), int(flush_bytes), steps, kern))
        return list(steps)[:int(n)], list(kern)

    def launches_per_apply(self) -> int:
        return int(self._lib.nfs_launches_per_apply(self._h))


def intensity_correction(sens_full, vox_index, device: int = 0) -> np.ndarray:
    """Device j = 1/sqrt(sum_c |S|^2) of the voxels `vox_index` (nfs/sensmaps.py:145-152)."""
    lib = load_library()
    full = _c128(sens_full)
    idx = np.ascontiguousarray(vox_index, dtype=np.int64)
    if full.ndim != 2:
        raise EngineError("sensitivity maps must be (L, coils)")
    out = np.empty(idx.size)
    _check(lib.nfs_intensity_correction(int(device), _dp(full.view(np.float64)), int(full.shape[0]),
                                        int(full.shape[1]), idx.ctypes.data_as(ctypes.POINTER(_c_i64)),
                                        int(idx.size), _dp(out)))
    return out


class SharedComm:
    """One NCCL communicator per rank, shared by every plan of the process (nfs_comm_create)."""

    def __init__(self, unique_id: bytes, rank: int, world: int, device: int):
        lib = load_library()
        h = _c_void_p()
        _check(lib.nfs_comm_create(unique_id, int(rank), int(world), int(device), ctypes.byref(h)))
        self._lib, self.handle, self.rank, self.world, self.device = lib, h, int(rank), int(world), int(device)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.nfs_comm_destroy(self.handle)
            self.handle = None
