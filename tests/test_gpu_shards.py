"""Sample sharding composes (nfs/engine.py:219-222): the per-rank plans of the
multi-GPU path, built exactly as engine._make_plan builds them (contiguous shard_rows of the
temporal table and of sigma, replicated spatial table and S'), sum to the unsharded operator.

Only one GPU exists in this run, so the shards run one after another on cuda:0 in one process
(no collective); what the NCCL all-reduce adds on N GPUs is this sum.  FP64: <= 1e-12 relative
and bit-stable across repeats; the fast modes: within their operator tolerance (their chunk
partition differs between a shard and the whole, so the rounding differs).
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

from paper_2604_09233_b200 import engine, simulate  # noqa: E402
from paper_2604_09233_b200._native import Plan  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def _plan(prob, lo, hi, prec):
    plan = Plan(hi - lo, prob.spatial.shape[1], prob.sens.shape[1], prob.spatial.shape[0], prec)
    plan.set_tables(prob.temporal[lo:hi], prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    return plan


def _sharded(prob, world, prec, fn):
    k = prob.temporal.shape[0]
    out = 0
    for r in range(world):
        lo, hi = engine.shard_rows(k, r, world)
        plan = _plan(prob, lo, hi, prec)
        try:
            out = out + fn(plan, lo, hi)
        finally:
            plan.close()
    return out


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_sum_to_unsharded_fp64(world):
    g = golden("config_a")
    prob = simulate.make_problem("A_mask")
    rng = np.random.default_rng(3)
    p = rng.standard_normal(prob.spatial.shape[1]) + 1j * rng.standard_normal(prob.spatial.shape[1])
    sigma = g["sigma"]
    k = prob.temporal.shape[0]
    whole = _plan(prob, 0, k, "fp64")
    try:
        ehe, eh = whole.apply_EHE(p), whole.apply_EH(sigma)
    finally:
        whole.close()
    s_ehe = _sharded(prob, world, "fp64", lambda pl, lo, hi: pl.apply_EHE(p))
    s_eh = _sharded(prob, world, "fp64", lambda pl, lo, hi: pl.apply_EH(sigma[lo:hi]))
    assert rel(s_ehe, ehe) < 1e-12
    assert rel(s_eh, eh) < 1e-12
    again = _sharded(prob, world, "fp64", lambda pl, lo, hi: pl.apply_EHE(p))
    assert np.array_equal(again, s_ehe)          # deterministic: bit-identical repeats


@pytest.mark.parametrize("prec", ["f16x3", "fp32"])
def test_shards_sum_to_unsharded_fast_modes(prec):
    prob = simulate.make_problem("B", scale=2)    # 128^2, K = 16,384: real split-K launches
    rng = np.random.default_rng(4)
    p = rng.standard_normal(prob.spatial.shape[1]) + 1j * rng.standard_normal(prob.spatial.shape[1])
    k = prob.temporal.shape[0]
    ref = _plan(prob, 0, k, "fp64")
    try:
        exact = ref.apply_EHE(p)
    finally:
        ref.close()
    s = _sharded(prob, 4, prec, lambda pl, lo, hi: pl.apply_EHE(p))
    assert rel(s, exact) < 2e-5
    again = _sharded(prob, 4, prec, lambda pl, lo, hi: pl.apply_EHE(p))
    assert np.array_equal(again, s)


def test_sharded_cg_matches_unsharded_fp64():
    """The CG every rank runs after the all-reduce, emulated with the shard sum on the host,
    tracks the unsharded device CG: the composition is exact enough for FP64 parity."""
    g = golden("engine8")
    from oracle import nfs_oracle as orc   # the CG recurrence (checker only)
    from paper_2604_09233_b200.core import Grid
    sigma, spatial, temporal, sens = g["sigma"], g["spatial"], g["temporal"], g["sens"]
    k, l = temporal.shape[0], spatial.shape[1]
    plans = []
    for r in range(3):
        lo, hi = engine.shard_rows(k, r, 3)
        pl = Plan(hi - lo, l, sens.shape[1], spatial.shape[0], "fp64")
        pl.set_tables(temporal[lo:hi], spatial)
        pl.set_sens(sens)
        plans.append((pl, lo, hi))
    try:
        ehe = lambda v: sum(pl.apply_EHE(v) for pl, _, _ in plans)   # noqa: E731
        p0 = sum(pl.apply_EH(sigma[lo:hi]) for pl, lo, hi in plans)
        rho = orc._cg(p0, ehe, 15, orc.OracleLog(), None)
    finally:
        for pl, _, _ in plans:
            pl.close()
    img, _ = engine.recon_full(engine.EncodingInputs(
        sigma=sigma, spatial=spatial, temporal=temporal, sens=sens, intensity=np.ones(l), kfilter=None,
        mask_r=np.ones(l, bool), grid=Grid((8, 8, 1), (0.08, 0.08, 0.002)), n_iter=15), precision="fp64")
    assert rel(rho, img.values) < 1e-10
    assert rel(rho, g["full_values"]) < 1e-10
