"""CPU checks of the boundary: the C-ABI library loads and exports every symbol the header
declares, the ctypes binding matches the header, and the Python shim validates like the
reference (no GPU needed, no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nfs_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nfs_[a-zA-Z_0-9]+)\s*\(", text)) - {"nfs_iter_callback"})


def test_library_exports_header_symbols():
    from paper_2604_09233_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert lib.nfs_version and ctypes.cast(lib.nfs_version, ctypes.c_void_p).value


def test_binding_matches_header():
    from paper_2604_09233_b200._native import SIGNATURES
    assert sorted(SIGNATURES) == header_functions()


def test_binding_loads_and_reports_version():
    from paper_2604_09233_b200 import _native
    lib = _native.load_library()
    assert lib.nfs_version().decode().startswith("nfs_b200")


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2604_09233_b200._native import Plan
    from paper_2604_09233_b200.errors import EngineError
    with pytest.raises(EngineError):
        Plan(10, 10, 2, 3, "fp32")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2604_09233_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|import_module\(.oracle|nfs_oracle",
                                     src, flags=re.M), f


def test_encoding_inputs_validation():
    from paper_2604_09233_b200 import EncodingInputs, EngineError, Grid
    grid = Grid((8, 8, 1), (0.08, 0.08, 0.002))
    sens = np.ones((64, 3), complex)
    spatial = np.zeros((3, 64))
    temporal = np.zeros((60, 3))

    def mk(sigma, **kw):
        args = dict(sigma=sigma, spatial=spatial, temporal=temporal, sens=sens,
                    intensity=np.ones(64), kfilter=None, mask_r=np.ones(64, bool), grid=grid,
                    n_iter=1)
        args.update(kw)
        return EncodingInputs(**args)

    with pytest.raises(EngineError):
        mk(np.zeros((61, 3), complex))
    with pytest.raises(EngineError):
        mk(np.zeros((60, 2), complex))
    mask = np.ones(64, bool)
    mask[0] = False
    with pytest.raises(EngineError):
        mk(np.zeros((60, 3), complex), mask_r=mask)
    for starts in ([1, 60], [0, 59], [0, 30, 30, 60]):
        with pytest.raises(EngineError):
            mk(np.zeros((60, 3), complex), block_starts=np.array(starts))
    ok = mk(np.zeros((60, 3), complex), block_starts=[0, 30, 60])
    assert ok.n_samples == 60 and ok.n_voxels == 64


def test_build_bases_matches_oracle():
    from oracle import nfs_oracle as orc
    from paper_2604_09233_b200 import Grid, build_bases
    from paper_2604_09233_b200.engine import EngineError
    rng = np.random.default_rng(1)
    for dims, order, nterm in (((8, 8, 1), 1, 2), ((6, 6, 4), 2, 8), ((6, 6, 4), 3, 15)):
        grid = Grid(dims, (0.1, 0.1, 0.05))
        mask = rng.random(grid.nvox) > 0.3
        b0 = rng.standard_normal(grid.nvox)
        t = np.linspace(0, 0.01, 40)
        terms = rng.standard_normal((40, nterm))
        s1, t1 = build_bases(b0, mask, grid, t, terms, order=order)
        s2, t2 = orc.build_bases(b0, mask, dims, grid.fov_m, t, terms, order=order)
        assert np.array_equal(s1, s2) and np.array_equal(t1, t2)
    with pytest.raises(EngineError):
        build_bases(np.zeros(64), np.ones(64, bool), Grid((8, 8, 1), (0.1, 0.1, 0.1)),
                    np.zeros(40), np.zeros((40, 2)), order=2)


def test_choose_block_starts_and_sharding():
    from oracle import nfs_oracle as orc
    from paper_2604_09233_b200.engine import choose_block_starts, shard_rows
    for n, v, b in ((1000, 50, 50 * 16 * 64), (5, 100, 1), (100, 10, 10**9), (7, 3, 100)):
        assert np.array_equal(choose_block_starts(n, v, b), orc.choose_block_starts(n, v, b))
    for n in (0, 1, 7, 65536, 299648):
        for w in (1, 2, 3, 8):
            spans = [shard_rows(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_header_is_plain_c_and_links(tmp_path):
    """The ABI is usable from plain C (what a cgo / JNI / N-API shim would compile against):
    the header compiles as C99 and a C program links against the built library (no GPU calls;
    it only queries the version string)."""
    import shutil
    import subprocess
    from paper_2604_09233_b200 import build
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib_path = build.build()
    src = tmp_path / "abi.c"
    src.write_text('#include <stdio.h>\n#include "nfs_b200.h"\n'
                   "int main(void) { nfs_plan* p = 0; (void)p; puts(nfs_version()); return 0; }\n")
    exe = tmp_path / "abi"
    subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                    lib_path, "-o", str(exe), f"-Wl,-rpath,{os.path.dirname(lib_path)}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert out.strip()


def test_dataset_samples_handle_host_side(tmp_path):
    """engine.DatasetSamples reads the reference's dataset manifest (nfs/core.py:292-328) and
    loads the whole array like Dataset.load_array when materialised (no GPU needed)."""
    import json
    from paper_2604_09233_b200 import engine
    sig = (np.arange(12) + 1j * np.arange(12)[::-1]).reshape(6, 2)
    sig.astype("<c16").tofile(tmp_path / "sigma.c128")
    (tmp_path / "manifest.json").write_text(json.dumps(
        {"version": 1, "arrays": {"sigma": {"file": "sigma.c128", "dtype": "c128", "shape": [6, 2]}}}))
    h = engine.DatasetSamples(tmp_path)
    assert h.shape == (6, 2) and h.ndim == 2
    assert np.array_equal(np.asarray(h), sig)
    (tmp_path / "manifest.json").write_text(json.dumps(
        {"version": 1, "arrays": {"sigma": {"file": "sigma.c128", "dtype": "c128", "shape": [7, 2]}}}))
    with pytest.raises(engine.EngineError):
        engine.DatasetSamples(tmp_path)
