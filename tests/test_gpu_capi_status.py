"""The C ABI's status codes, called directly through ctypes the way a maintainer's binding would
(include/nfs_b200.h; mapped onto EngineError / MemoryBudgetError by the Python shim)."""
import ctypes

import numpy as np
import pytest

from paper_2604_09233_b200 import _native

pytestmark = pytest.mark.gpu

OK, INVALID, NONFINITE = 0, 1, 2


@pytest.fixture(scope="module")
def lib():
    return _native.load_library()


def _create(lib, K, L, G, P1, prec, dev=0):
    h = ctypes.c_void_p()
    st = lib.nfs_plan_create(ctypes.byref(h), K, L, G, P1, prec, dev)
    return st, h


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def test_create_rejects_bad_arguments(lib):
    st, h = _create(lib, 100, 50, 4, 33, 1)            # more than 32 basis terms
    assert st == INVALID and not h.value and b"32" in lib.nfs_last_error()
    st, _ = _create(lib, 100, 50, 4, 3, 9)             # unknown precision
    assert st == INVALID
    st, _ = _create(lib, 100, 50, 4, 3, 1, dev=999)    # no such device
    assert st == INVALID
    lib.nfs_plan_destroy(None)                        # destroying NULL is a no-op


@pytest.mark.parametrize("prec", [0, 1, 3])
def test_call_order_and_data_errors(lib, prec):
    K, L, G, P1 = 300, 120, 4, 3
    st, h = _create(lib, K, L, G, P1, prec)
    assert st == OK, lib.nfs_last_error()
    try:
        p = np.zeros(2 * L)
        q = np.zeros(2 * L)
        assert lib.nfs_apply_EHE(h, _dp(p), _dp(q)) == INVALID            # no tables / sens yet
        assert lib.nfs_set_tables(h, None, None) == INVALID
        rng = np.random.default_rng(0)
        temporal = np.ascontiguousarray(rng.standard_normal((K, P1)))
        spatial = np.ascontiguousarray(rng.standard_normal((P1, L)))
        sens = rng.standard_normal((L, 2 * G))
        assert lib.nfs_set_tables(h, _dp(temporal), _dp(spatial)) == OK
        assert lib.nfs_set_sens(h, _dp(sens), None) == OK
        rho = np.zeros(2 * L)
        res = np.zeros(4)
        sol = np.zeros(4)
        done = ctypes.c_int32()
        tim = np.zeros(6)
        # CG before the samples are set
        assert lib.nfs_cg_solve(h, 4, _native.CALLBACK(), None, _dp(rho), _dp(res), _dp(sol),
                                ctypes.byref(done), _dp(tim)) == INVALID
        sigma = rng.standard_normal((K, 2 * G))
        sigma[7, 3] = np.nan
        assert lib.nfs_set_samples(h, _dp(sigma)) == NONFINITE
        sigma[7, 3] = 0.0
        assert lib.nfs_set_samples(h, _dp(sigma)) == OK
        assert lib.nfs_cg_solve(h, 4, _native.CALLBACK(), None, _dp(rho), _dp(res), _dp(sol),
                                ctypes.byref(done), _dp(tim)) == OK
        assert done.value == 4 and np.all(np.isfinite(rho)) and res[0] > 0
    finally:
        lib.nfs_plan_destroy(h)
