"""Multi-rank sample sharding on CPU (world_size 2, gloo): the decomposition the GPU path uses.

Each rank holds a contiguous shard of the readout samples (engine.shard_rows), applies its
shard's E_r^H E_r, and the adjoint images are all-reduced (sum) once per CG iteration; every
rank then runs the identical CG update.  The result must equal the single-process oracle CG
(nfs/engine.py:154-178) to rounding, and every rank must hold the same image.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nfs_oracle as orc
    from paper_2604_09233_b200.engine import shard_rows

    g = golden("engine8")
    sigma, spatial, temporal, sens = g["sigma"], g["spatial"], g["temporal"], g["sens"]
    lo, hi = shard_rows(temporal.shape[0], rank, world)
    ph = orc.phase_block(temporal[lo:hi], spatial)

    def allreduce(v):
        t = torch.from_numpy(np.ascontiguousarray(v).view(np.float64).copy())
        dist.all_reduce(t)
        return t.numpy().view(np.complex128)

    def ehe(p):   # per-iteration exchange: one all-reduce of the adjoint image
        return allreduce(orc.apply_EH(orc.apply_E(p, sens, ph), sens, ph))

    p0 = allreduce(orc.apply_EH(sigma[lo:hi], sens, ph))
    log = orc.OracleLog()
    rho = orc._cg(p0, ehe, 15, log, None)
    np.save(os.path.join(out_dir, f"rho{rank}.npy"), rho)
    np.save(os.path.join(out_dir, f"res{rank}.npy"), np.array(log.residual_norms))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sample_sharded_cg_matches_single_process(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    from oracle import nfs_oracle as orc

    g = golden("engine8")
    ref, ref_log = orc.recon_full(g["sigma"], g["spatial"], g["temporal"], g["sens"], np.ones(64), 15)
    rhos = [np.load(tmp_path / f"rho{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(rhos[r], rhos[0])          # identical on every rank
    assert np.linalg.norm(rhos[0] - ref) / np.linalg.norm(ref) < 1e-10
    assert np.allclose(np.load(tmp_path / "res0.npy"), ref_log.residual_norms, rtol=1e-8)
    assert np.allclose(rhos[0], g["full_values"], atol=1e-10)


def _slices_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_09233_b200 import engine

    calls = []

    def fake_recon(inputs, callback, precision, shard):   # the GPU solve, replaced on CPU
        assert shard is False and callback is None
        calls.append(int(inputs))
        return ("image", int(inputs), rank), ("log", int(inputs))

    engine._recon_full = fake_recon
    n = 7

    class Fake(int):   # stands in for EncodingInputs (size checks only)
        sigma, spatial = np.zeros((3, 1)), np.zeros((1, 5))

    out = engine.recon_slices([Fake(i) for i in range(n)])
    np.save(os.path.join(out_dir, f"slices{rank}.npy"),
            np.array([[r[0][1], r[0][2], r[1][1]] for r in out]))
    np.save(os.path.join(out_dir, f"calls{rank}.npy"), np.array(calls))
    dist.destroy_process_group()


def test_recon_slices_replicas_without_collective(tmp_path):
    """slice i is solved on rank i mod world (no collective in the solve)
    and every rank receives all results in slice order."""
    world = 2
    port = _free_port()
    mp.spawn(_slices_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        got = np.load(tmp_path / f"slices{r}.npy")
        assert np.array_equal(got[:, 0], np.arange(7)) and np.array_equal(got[:, 2], np.arange(7))
        assert np.array_equal(got[:, 1], np.arange(7) % world)      # solved by rank i mod world
        assert np.array_equal(np.load(tmp_path / f"calls{r}.npy"), np.arange(r, 7, world))


def _slices_fail_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_09233_b200 import engine

    def fake_recon(inputs, callback, precision, shard):
        if int(inputs) == 3:   # slice 3 (rank 1) fails inside its solve, e.g. non-finite data
            raise engine.EngineError("raw data contains non-finite values")
        return ("image", int(inputs), rank), ("log", int(inputs))

    engine._recon_full = fake_recon

    class Fake(int):
        sigma, spatial = np.zeros((3, 1)), np.zeros((1, 5))

    try:
        engine.recon_slices([Fake(i) for i in range(6)])
        msg = "no error"
    except engine.EngineError as exc:
        msg = f"{type(exc).__name__}: {exc}"
    with open(os.path.join(out_dir, f"err{rank}.txt"), "w") as f:
        f.write(msg)
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_recon_slices_failure_reaches_every_rank(tmp_path):
    """A slice failing on one rank must not leave the others blocked in the result gather
    (ADVICE r1): every rank raises, the owner its own exception, the others an EngineError
    naming the slice."""
    world = 2
    port = _free_port()
    mp.spawn(_slices_fail_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    e0 = (tmp_path / "err0.txt").read_text()
    e1 = (tmp_path / "err1.txt").read_text()
    assert e1 == "EngineError: raw data contains non-finite values"
    assert e0.startswith("EngineError: slice 3 failed on another rank"), e0
