"""Race detection by timing perturbation (compute-sanitizer is closed on this GPU pool).

The f16x3 kernel is a warp-specialised pipeline: 12 generator warps in three chunk groups, two
contraction issuers, a phase issuer, a producer and four drain warps hand TMEM and shared-memory
stages to each other through mbarriers, in 2-CTA multicast clusters.  A hand-off that relies on
the usual timing instead of a barrier shows up only when the roles interleave differently.  This
test builds the same kernel with `-DNFS_TCI_JITTER=1` (the TF32x3 kernel: `-DNFS_TC_JITTER=1`) -- pseudo-random sleeps of up to ~2 us at one
in four hand-offs of every role (`jitter()` in csrc/nfs_tci.cu; the product build compiles it to
nothing, its SASS is unchanged) -- and requires the operators and a short CG solve to be
bit-identical to the product library's.  An earlier version of the issuers' A-stage wait (a parity
probe latched before the D-buffer wait) fails it: with the jitter, configs A and B
deadlock (a subprocess timeout here) -- `-DNFS_TCI_SPIN3_LATCH` rebuilds that version.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("A_mask", 1), ("B", 8), ("D", 4), ("B", 1)]   # NC = 8 / small grids / 3D / full launch shape
CASES_TC = [("A_mask", 1), ("B", 8)]                     # the TF32x3 kernel (csrc/nfs_tc.cu), same idea


def _build(name, flag, src):
    import shutil
    if shutil.which("nvcc") is None:
        pytest.skip("nvcc not on PATH: the race-detection variant cannot be built here")
    env = dict(os.environ, VAR_SRC=src)
    r = subprocess.run(["bash", os.path.join(ROOT, "tools", "build_variant.sh"), name, flag],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    path = os.path.join(ROOT, r.stdout.strip().splitlines()[-1])
    assert os.path.exists(path)
    return path


@pytest.fixture(scope="module")
def jitter_lib():
    return _build("jitter", "-DNFS_TCI_JITTER=1", "nfs_tci")


@pytest.fixture(scope="module")
def jitter_lib_tc():
    return _build("jitter_tc", "-DNFS_TC_JITTER=1", "nfs_tc")


def _run(lib, config, scale, out, precision="f16x3"):
    env = dict(os.environ)
    if lib:
        env["NFS_B200_LIB"] = lib
    else:
        env.pop("NFS_B200_LIB", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab_check.py"), "--config", config,
                        "--scale", str(scale), "--out", out, "--precision", precision], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=180)   # a few seconds when correct; a deadlocked pipeline never returns
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("config,scale", CASES)
def test_jittered_schedule_is_bit_identical(jitter_lib, tmp_path, config, scale):
    ref = _run(None, config, scale, str(tmp_path / "product.npz"))
    jit = _run(jitter_lib, config, scale, str(tmp_path / "jitter.npz"))
    for k in ("y_sha", "q_sha", "rho_sha", "res"):
        assert np.array_equal(ref[k], jit[k]), f"{config} x{scale}: {k} differs under a perturbed schedule"


@pytest.mark.parametrize("config,scale", CASES_TC)
def test_jittered_schedule_is_bit_identical_tf32x3(jitter_lib_tc, tmp_path, config, scale):
    ref = _run(None, config, scale, str(tmp_path / "product.npz"), "tf32x3")
    jit = _run(jitter_lib_tc, config, scale, str(tmp_path / "jitter.npz"), "tf32x3")
    for k in ("y_sha", "q_sha", "rho_sha", "res"):
        assert np.array_equal(ref[k], jit[k]), f"tf32x3 {config} x{scale}: {k} differs under a perturbed schedule"
